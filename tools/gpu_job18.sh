# float2 intrinsics (-37% SASS on fp32), clamped tail loads, ramped host chunks:
# GPU tests, bench, sweeps, sustained A/B.
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.json
timeout 400 python tools/sweep.py --json gpurun_out/sweep_fwd.json > gpurun_out/sweep_fwd.log 2>&1
cat gpurun_out/sweep_fwd.log | tail -25
timeout 300 python tools/sustained.py 1024 single 65536 0,1,4,7 --secs 4 --rounds 2 > gpurun_out/sus_1024s.json 2>&1
timeout 300 python tools/sustained.py 2048 single 65536 0,3,4,5 --secs 4 --rounds 2 > gpurun_out/sus_2048s.json 2>&1
timeout 300 python tools/sustained.py 2048 double 32768 0,1,3,4 --secs 4 --rounds 2 > gpurun_out/sus_2048d.json 2>&1
timeout 300 python tools/sustained.py 1024 double 65536 0,1,3,4 --secs 4 --rounds 2 > gpurun_out/sus_1024d.json 2>&1
timeout 300 python tools/sustained.py 512 single 262144 0,1,2 --secs 4 --rounds 2 > gpurun_out/sus_512s.json 2>&1
cat gpurun_out/sus_*.json
