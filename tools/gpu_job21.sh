# Per-variant smem carveout (50% for LDG variants): tests, all-variant sweep, sustained A/B.
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
timeout 600 python tools/sweep.py --all-variants --json gpurun_out/sweep_all.json > gpurun_out/sweep_all.log 2>&1
timeout 300 python tools/sustained.py 1024 single 65536 0,1,2,4 --secs 4 --rounds 2 > gpurun_out/sus_1024s.json 2>&1
timeout 300 python tools/sustained.py 2048 single 65536 0,1,4,6 --secs 4 --rounds 2 > gpurun_out/sus_2048s.json 2>&1
timeout 300 python tools/sustained.py 2048 double 32768 0,1,4 --secs 4 --rounds 2 > gpurun_out/sus_2048d.json 2>&1
timeout 300 python tools/sustained.py 1024 double 65536 0,1,4 --secs 4 --rounds 2 > gpurun_out/sus_1024d.json 2>&1
cat gpurun_out/sus_*.json
