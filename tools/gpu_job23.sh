# Persistent pipelined TMA kernel (loader 2): tests, sanitizers on it, sweep, sustained A/B.
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick --loader 2 > gpurun_out/san_race_pipe.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_run.py --quick --loader 2 > gpurun_out/san_sync_pipe.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py --loader 2 > gpurun_out/san_mem_pipe.txt 2>&1
tail -n 3 gpurun_out/san_*_pipe.txt
timeout 600 python tools/sweep.py --all-variants --cool 0.5 --n 512,1024,2048 --json gpurun_out/sweep_pipe.json > gpurun_out/sweep_pipe.log 2>&1
timeout 300 python tools/sustained.py 1024 single 65536 0,8,9,10 --secs 4 --rounds 2 > gpurun_out/sus_1024s.json 2>&1
timeout 300 python tools/sustained.py 2048 single 65536 0,4,7,8 --secs 4 --rounds 2 > gpurun_out/sus_2048s.json 2>&1
timeout 300 python tools/sustained.py 2048 double 32768 0,4,5,6 --secs 4 --rounds 2 > gpurun_out/sus_2048d.json 2>&1
timeout 300 python tools/sustained.py 1024 double 65536 1,5,6 --secs 4 --rounds 2 > gpurun_out/sus_1024d.json 2>&1
timeout 300 python tools/sustained.py 512 double 131072 0,4 --secs 4 --rounds 2 > gpurun_out/sus_512d.json 2>&1
timeout 300 python tools/sustained.py 512 single 262144 0,3 --secs 4 --rounds 2 > gpurun_out/sus_512s.json 2>&1
cat gpurun_out/sus_*.json
