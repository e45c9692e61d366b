set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/sweep.py --all-variants --json gpurun_out/sweep_fwd.json > gpurun_out/sweep_fwd.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -3 gpurun_out/pytest_gpu.log
