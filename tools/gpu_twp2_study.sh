set -x
python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -4
python tools/variant_accuracy.py gpurun_out/r02_variant_accuracy.json > /dev/null 2>&1
python tools/sweep.py --all-variants --cool 0.3 --n 64,128,256,512,1024,2048 --json gpurun_out/r02_sweep_variants.json > /dev/null 2>&1
for spec in "2048 single 65536 copy,0,7" "1024 single 131072 copy,0,9" "2048 double 32768 copy,0,6" "1024 double 65536 copy,0,5"; do
  python tools/sustained.py $spec --secs 4 --rounds 2 >> gpurun_out/r02_sustained_twp2.jsonl 2>&1
done
