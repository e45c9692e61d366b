# Round-2 loader / twiddle variant study for the sustained-load gap (fp64 N>=1024, fp32 N=2048).
set -x
python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "all_kernel_variants" 2>&1 | tail -2
python tools/sweep.py --all-variants --cool 0.3 --n 1024,2048 --json gpurun_out/r02_sweep_study.json > /dev/null 2>&1
for spec in "2048 double 32768 copy,0,4,7,8" "1024 double 65536 copy,0,4,6,7" "2048 single 65536 copy,0,5,8"; do
  python tools/sustained.py $spec --secs 4 --rounds 2 >> gpurun_out/r02_sustained_study.jsonl 2>&1
done
