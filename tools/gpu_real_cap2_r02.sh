set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for round in 1 2 3; do
  NS=512 VARIANT_SINGLE_512=0 python tools/real_input_probe.py 2>&1 | grep single
  NS=512 VARIANT_SINGLE_512=6 python tools/real_input_probe.py 2>&1 | grep single
  NS=2048 python tools/real_input_probe.py 2>&1 | grep single
done
timeout 300 python tools/sustained.py 2048 single 65536 copy,0 --secs 3 --rounds 1 2>&1 | tail -1
