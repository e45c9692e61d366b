set -x
python tools/pcie_probe.py > gpurun_out/pcie.json 2>&1
for cfg in "double 2048 0" "double 2048 2" "double 1024 0" "double 1024 3" "single 2048 0"; do
  set -- $cfg
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:stockham -s 2 -c 1 \
     -o gpurun_out/prof2_${1}_${2}_v${3} python tools/sweep.py --prec $1 --n $2 --iters 1 --warmup 2 --variant $3 > /dev/null 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 10 > gpurun_out/bench_c2b.json 2>&1
