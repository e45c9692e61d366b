# fp64 N=2048: split re/im exchange (LAYOUT 3, LDG loader, variant 12) and LDG with a 75 % carveout
# (variant 13) against the default R16 bulk-TMA kernel (variant 0): parity, burst, sustained, real input.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "variant" 2>&1 | tail -3
python tools/sweep.py --prec double --n 2048 --all-variants --cool 0.3 2>&1 | tail -20
python tools/sustained.py 2048 double 131072 copy,0,12,13 --secs 4 --rounds 3 2>&1 | tail -2
VARIANT_DOUBLE_2048=12 NS=2048 python tools/real_input_probe.py 2>&1 | grep double
VARIANT_DOUBLE_2048=13 NS=2048 python tools/real_input_probe.py 2>&1 | grep double
NS=2048 python tools/real_input_probe.py 2>&1 | grep double
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c4_v12 python tools/launch_variant.py 2048 double 131072 12 > gpurun_out/ncu_c4_v12.log 2>&1
tail -3 gpurun_out/ncu_c4_v12.log
