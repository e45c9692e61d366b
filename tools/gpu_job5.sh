set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/sweep.py --all-variants --n 128,256,512,1024,2048 --json gpurun_out/sweep_fwd5.json > gpurun_out/sweep_fwd5.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
