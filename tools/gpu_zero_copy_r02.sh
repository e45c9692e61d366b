# Zero-copy small-call host path: GPU API tests, A/B against the copy-engine path, and the
# paper section 6.1 host latency protocol with the new default.
set -x
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_abi.py -q -p no:cacheprovider 2>&1 | tail -3
SFFT_ZERO_COPY_BYTES=0 python tools/zero_copy_probe.py > gpurun_out/zc0.jsonl 2>&1
python tools/zero_copy_probe.py > gpurun_out/zc1.jsonl 2>&1
timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --records gpurun_out/latency_host_records.csv --summary gpurun_out/latency_host.json > gpurun_out/latency_host.txt 2>&1
SFFT_ZERO_COPY_BYTES=0 timeout 600 python -m paper_2203_09384_b200 bench --lengths 8:2048:pow2 --iterations 1000 --warmup 1 --summary gpurun_out/latency_host_copies.json > gpurun_out/latency_host_copies.txt 2>&1
python - <<PY
import json
a=json.load(open("gpurun_out/latency_host_copies.json"))["summaries"]; b=json.load(open("gpurun_out/latency_host.json"))["summaries"]
for x,y in zip(a,b): print(x["length"], "copies", round(x["optimal_us"],1), round(x["mean_us"],1), "zero-copy", round(y["optimal_us"],1), round(y["mean_us"],1))
PY
