# Round-2 study 3: candidate defaults (wide radix + bulk TMA, real-input capable) vs round-1 defaults.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "all_kernel_variants" 2>&1 | tail -2
python tools/variant_accuracy.py gpurun_out/r02_variant_accuracy3.json > /dev/null 2>&1
NS=1024,2048 python tools/real_input_probe.py > gpurun_out/r02_real_default.jsonl 2>&1
NS=1024,2048 VARIANT_SINGLE_2048=13 VARIANT_DOUBLE_1024=11 VARIANT_DOUBLE_2048=11 python tools/real_input_probe.py > gpurun_out/r02_real_candidates.jsonl 2>&1
NS=1024,2048 VARIANT_SINGLE_2048=14 python tools/real_input_probe.py > gpurun_out/r02_real_candidates14.jsonl 2>&1
python tools/sweep.py --all-variants --cool 0.3 --n 1024,2048 --json gpurun_out/r02_sweep_study3.json > /dev/null 2>&1
for spec in "2048 single 65536 copy,0,13,14" "1024 double 65536 copy,0,11" "2048 double 32768 copy,0,11"; do
  python tools/sustained.py $spec --secs 4 --rounds 3 >> gpurun_out/r02_sustained_study3.jsonl 2>&1
done
