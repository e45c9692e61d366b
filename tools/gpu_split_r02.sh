# Host pipeline: mid-size calls cut into several chunks (pinned: 4 up to 32 MiB, else 8; pageable: 4;
# >= 2 MiB each) vs one chunk per 32 MiB (SFFT_HOST_SPLIT=1); GPU suite for the host paths.
set -x
timeout 600 python -m pytest tests/test_gpu_api.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_config_parity.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do
  SFFT_HOST_SPLIT=1 timeout 300 python tools/e2e_size_probe.py
  timeout 300 python tools/e2e_size_probe.py
done
