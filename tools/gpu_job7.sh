set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
SFFT_BENCH_DIST_BACKEND=gloo SFFT_BENCH_DEVICE=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err
timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --records gpurun_out/latency_host_records.csv --summary gpurun_out/latency_host.json > gpurun_out/latency_host.txt 2>&1
timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --device cuda:0 --summary gpurun_out/latency_dev.json > gpurun_out/latency_dev.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log
