# fp64 N=2048: split-radix-2 two-warp kernel (split2) vs the R16 default.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -q -p no:cacheprovider -k "all_kernel_variants or every_real_capable" 2>&1 | tail -2
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --loader 1 2>&1 | tail -2
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py --quick --loader 1 2>&1 | tail -2
python tools/sweep.py --all-variants --cool 0.3 --n 2048 --prec double --json gpurun_out/r02_sweep_split2.json > /dev/null 2>&1
NS=2048 VARIANT_DOUBLE_2048=11 python tools/real_input_probe.py 2>&1 | grep double
NS=2048 python tools/real_input_probe.py 2>&1 | grep double
python tools/sustained.py 2048 double 32768 copy,0,9,11 --secs 4 --rounds 3 > gpurun_out/r02_sustained_split2.jsonl 2>&1
