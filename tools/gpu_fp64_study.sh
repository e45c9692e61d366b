# fp64 N=2048: what limits the SM side?  FP64 pipe rate probe + one ncu --set full capture of the c4 kernel.
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/fp64_probe tools/probe/fp64_probe.cu && ./tools/probe/fp64_probe
B="python bench.py --steps 4 --warmup 3 --no-cpu --no-extras --e2e-steps 1 --no-check"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stockham -s 3 -c 1 -o gpurun_out/prof_c4b $B --config c4 > gpurun_out/ncu_c4b.log 2>&1
ls -la gpurun_out
