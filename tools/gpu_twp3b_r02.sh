# TWP 3 for fp64 N=2048 (variant 14): accuracy, a second sustained A/B, ncu capture.
set -x
python tools/variant_accuracy.py 2>&1 | grep -E '"prec": "double", "n": 2048'
python tools/sustained.py 2048 double 131072 copy,0,14 --secs 4 --rounds 3 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c4_v14 python tools/launch_variant.py 2048 double 131072 14 > gpurun_out/ncu_c4_v14.log 2>&1
tail -2 gpurun_out/ncu_c4_v14.log
