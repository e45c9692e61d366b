# CUDA-graph replay of launch chains: after the capture-aware PDL switch (captured launches without
# programmatic dependent launch), vs eager; plus the graph tests and the eager latency path.
set -x
timeout 300 python -m pytest tests/test_gpu_api.py -m gpu -q -p no:cacheprovider -k "graph or chain or pdl or launch" 2>&1 | tail -2
timeout 300 python tools/graph_probe.py
timeout 300 python tools/graph_probe.py
timeout 300 python tools/latency_parts.py 2>&1 | tail -12
