timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/sweep.py --all-variants --n 256,1024,2048 --json gpurun_out/sweep_tma.json > gpurun_out/sweep_tma.log 2>&1
timeout 600 python tools/sweep.py --all-variants --n 256,1024,2048 --json gpurun_out/sweep_tma2.json > gpurun_out/sweep_tma2.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
