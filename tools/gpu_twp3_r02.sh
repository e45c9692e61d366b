# TWP 3 (one twiddle load per butterfly) for fp64 N=2048 (variant 14) and N=1024 (variant 10)
# against the defaults: parity, burst, sustained, real input.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "variant" 2>&1 | tail -3
python tools/sweep.py --prec double --n 1024,2048 --all-variants --cool 0.3 2>&1 | grep -E '"variant": (0|10|12|14),'
python tools/sustained.py 2048 double 131072 copy,0,14,12 --secs 4 --rounds 3 2>&1 | tail -1
python tools/sustained.py 1024 double 131072 copy,0,10 --secs 4 --rounds 3 2>&1 | tail -1
VARIANT_DOUBLE_2048=14 VARIANT_DOUBLE_1024=10 NS=1024,2048 python tools/real_input_probe.py 2>&1 | grep double
NS=1024,2048 python tools/real_input_probe.py 2>&1 | grep double
python tools/variant_accuracy.py 2>&1 | grep -E 'double.*(1024|2048)' | head
