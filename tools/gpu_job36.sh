# L2 bulk prefetch one resident wave ahead: tests, burst sweep, sustained vs copy.
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
timeout 600 python tools/sweep.py --all-variants --cool 0.3 --n 1024,2048 --json gpurun_out/sweep_pf.json > gpurun_out/sweep_pf.log 2>&1
timeout 300 python tools/sustained.py 1024 single 65536 copy,0,9,10 --secs 4 --rounds 2 > gpurun_out/pf_1024s.json 2>&1
timeout 300 python tools/sustained.py 2048 single 65536 copy,0,7,8 --secs 4 --rounds 2 > gpurun_out/pf_2048s.json 2>&1
timeout 300 python tools/sustained.py 2048 double 131072 copy,0,6,7 --secs 4 --rounds 2 > gpurun_out/pf_2048d.json 2>&1
timeout 300 python tools/sustained.py 1024 double 65536 copy,0,5,6 --secs 4 --rounds 2 > gpurun_out/pf_1024d.json 2>&1
cat gpurun_out/pf_*.json
