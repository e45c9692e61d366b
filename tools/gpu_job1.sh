set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 400 python tools/sweep.py --all-variants --json gpurun_out/sweep_fwd.json > gpurun_out/sweep_fwd.log 2>&1
timeout 300 python tools/sweep.py --dir inverse --json gpurun_out/sweep_inv.json > gpurun_out/sweep_inv.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 1 --no-check > gpurun_out/ncu_launch_run.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 4 --warmup 3 --no-cpu --e2e-steps 1 --no-check > gpurun_out/ncu_full_run.log 2>&1
ls -la gpurun_out
