# Row-swizzle layout (LAYOUT 2) for fp64 + fp64 non-finite prefilter: tests, sweeps, sustained, ncu c4.
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --all-variants --cool 0.5 --json gpurun_out/sweep_all.json > gpurun_out/sweep_all.log 2>&1
timeout 300 python tools/sustained.py 2048 double 32768 0,1,4 --secs 4 --rounds 2 > gpurun_out/sus_2048d.json 2>&1
timeout 300 python tools/sustained.py 1024 double 65536 0,1,4 --secs 4 --rounds 2 > gpurun_out/sus_1024d.json 2>&1
timeout 300 python tools/sustained.py 512 double 131072 0,1,3 --secs 4 --rounds 2 > gpurun_out/sus_512d.json 2>&1
cat gpurun_out/sus_*.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c4 python bench.py --config c4 --steps 4 --warmup 3 --no-cpu --e2e-steps 1 --no-check > gpurun_out/ncu_full_run_c4.log 2>&1
