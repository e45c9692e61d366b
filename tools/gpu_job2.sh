set -x
for cfg in "single 2048 0" "double 1024 0" "double 1024 1" "double 2048 0" "single 1024 0"; do
  set -- $cfg
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:stockham -s 2 -c 1 \
     -o gpurun_out/prof_${1}_${2}_v${3} python tools/sweep.py --prec $1 --n $2 --iters 1 --warmup 2 --variant $3 > gpurun_out/ncu_${1}_${2}_v${3}.log 2>&1
done
ls -la gpurun_out
