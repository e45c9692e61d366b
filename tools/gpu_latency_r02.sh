# paper section 6.1 latency protocol + execute() cost breakdown + vendor latency, same box.
set -x
python tools/latency_parts.py > gpurun_out/latency_parts.txt 2>&1
timeout 600 python tools/vs_cufft.py --latency --json gpurun_out/latency_vs_cufft.json > gpurun_out/latency_vs_cufft.log 2>&1
timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --records gpurun_out/latency_host_records.csv --summary gpurun_out/latency_host.json > gpurun_out/latency_host.txt 2>&1
timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --device cuda:0 --records gpurun_out/latency_dev_records.csv --summary gpurun_out/latency_dev.json > gpurun_out/latency_dev.txt 2>&1
