# Sustained (power-capped) sweep of the defaults for every N, plus the fp64 N=512 wide-radix candidates.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "all_kernel_variants" 2>&1 | tail -2
bash tools/sustained_sweep.sh > gpurun_out/r02_sustained_sweep.jsonl 2>&1
python tools/sustained.py 512 double 131072 copy,0,4,5,6 --secs 4 --rounds 3 > gpurun_out/r02_sustained_f64_512.jsonl 2>&1
python tools/sweep.py --all-variants --cool 0.3 --n 512 --prec double --json gpurun_out/r02_sweep_f64_512.json > /dev/null 2>&1
