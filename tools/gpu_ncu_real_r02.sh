# ncu of the real-input loaders at the weakest real-input points: fp32 N=2048 and fp64 N=2048 / 1024
set -x
for cfg in "2048 single 65536" "2048 double 32768" "1024 double 65536"; do
  set -- $cfg
  REAL=1 timeout 300 ncu --set full --clock-control none -k regex:"stockham" -s 2 -c 1 -o gpurun_out/prof_real_$1_$2 python tools/launch_variant.py $1 $2 $3 0 3 > gpurun_out/ncu_real_$1_$2.log 2>&1
  timeout 300 ncu --set full --clock-control none -k regex:"stockham" -s 2 -c 1 -o gpurun_out/prof_cplx_$1_$2 python tools/launch_variant.py $1 $2 $3 0 3 > gpurun_out/ncu_cplx_$1_$2.log 2>&1
done
ls gpurun_out/*.ncu-rep
