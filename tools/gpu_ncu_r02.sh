# ncu captures for round 2: c4 (fp64 N=2048, the kernel VERDICT r1 names), c2, and fp32 N=2048 (new TWP 2 default).
set -x
B="python bench.py --steps 4 --warmup 3 --no-cpu --no-extras --e2e-steps 1 --no-check"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c4 $B --config c4 > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c2 $B --config c2 > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_f2048 $B --n 2048 --precision single > gpurun_out/ncu_f2048.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 --no-check > gpurun_out/ncu_launch_run.log 2>&1
ls -la gpurun_out/
