# The round-1 experiments behind profiles/ (run on one B200 via gpurun; each
# line names the profile it produced).  tools/gpu_final.sh is the round-end
# measurement set (tests, bench lines, sweeps, accuracy, ncu, sanitizers).
set -x
# HBM ceiling: plain streaming kernels -> r01_hbm_ceiling_probe.txt
(cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe bw_probe.cu && ./bw_probe) > gpurun_out/hbm_ceiling_probe.txt 2>&1
# resident CTAs / L1-vs-shared carveout sweep -> r01_occ_probe.txt
(cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o occ_probe occ_probe.cu && ./occ_probe) > gpurun_out/occ_probe.txt 2>&1
# every compiled variant, burst -> r01_pipe_vs_resident.txt (with the sustained runs below)
timeout 900 python tools/sweep.py --all-variants --cool 0.3 --json gpurun_out/sweep_all.json > gpurun_out/sweep_all.log 2>&1
# power-capped steady state, kernels vs copy_ -> r01_sustained_*.jsonl
timeout 300 python tools/sustained.py 1024 single 65536 copy,0,1,2 --secs 4 --rounds 2 > gpurun_out/sus_1024s.json 2>&1
timeout 300 python tools/sustained.py 2048 double 131072 copy,0,1,4 --secs 4 --rounds 2 > gpurun_out/sus_2048d.json 2>&1
# HBM-filling fp64 N=2048 (BASELINE configs[3]) -> r01_bench_c4_fill_hbm.json
timeout 900 python bench.py --config c4 --fill-hbm 0.9 --steps 10 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/bench_c4_fill.json 2>&1
# vendor library comparison (throughput, latency) -> r01_vs_cufft.json, r01_latency_vs_cufft.json
timeout 800 python tools/vs_cufft.py --json gpurun_out/vs_cufft.json > gpurun_out/vs_cufft.log 2>&1
timeout 600 python tools/vs_cufft.py --latency --json gpurun_out/latency_vs_cufft.json > gpurun_out/latency_vs_cufft.log 2>&1
# paper §6.1 protocol -> r01_latency_{host,dev}.json + records
timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --records gpurun_out/latency_host_records.csv --summary gpurun_out/latency_host.json > gpurun_out/latency_host.txt 2>&1
timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --device cuda:0 --records gpurun_out/latency_dev_records.csv --summary gpurun_out/latency_dev.json > gpurun_out/latency_dev.txt 2>&1
# host link: pipeline vs free-running copies -> r01_e2e_link.jsonl; chunk/slot sweep -> r01_e2e_sweep.jsonl
for c in 8 32; do CHUNK_MB=$c SFFT_HOST_CHUNK_MB=$c timeout 120 python tools/e2e_link_probe.py; done > gpurun_out/e2e_link.jsonl 2>&1
for sl in 2 3 4; do for c in 16 32 64; do SFFT_HOST_SLOTS=$sl SFFT_HOST_CHUNK_MB=$c timeout 120 python tools/e2e_probe.py; done; done > gpurun_out/e2e_sweep.jsonl 2>&1
timeout 300 python tools/e2e_pageable.py > gpurun_out/e2e_pageable.json 2>&1
# N>1 bench path with 2 ranks sharing the one GPU -> r01_bench_c{2,5}_2ranks_1gpu*.json
SFFT_BENCH_DEVICE=0 SFFT_BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --no-cpu --steps 20 > gpurun_out/bench_2rank_1gpu.json 2>&1
