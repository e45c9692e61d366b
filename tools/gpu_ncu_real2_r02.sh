# ncu of the register-capped fp32 N=2048 real-input default (stockham_kernel_capped)
set -x
REAL=1 timeout 300 ncu --set full --clock-control none -k regex:"stockham" -s 2 -c 1 -o gpurun_out/prof_real_capped_2048 python tools/launch_variant.py 2048 single 65536 0 3 > gpurun_out/ncu_real_capped.log 2>&1
