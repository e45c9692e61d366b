set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --records gpurun_out/latency_host_records.csv --summary gpurun_out/latency_host.json > gpurun_out/latency_host.txt 2>&1
timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --device cuda:0 --records gpurun_out/latency_dev_records.csv --summary gpurun_out/latency_dev.json > gpurun_out/latency_dev.txt 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -3 gpurun_out/pytest_gpu.log
