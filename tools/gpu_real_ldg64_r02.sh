# fp64 N=2048 real input: the default bulk-TMA real loader vs per-thread LDG real loads on the same
# passes (variant 17), at the LDG carveout (50 %) and with the carveout lifted (SFFT_SMEM_CARVEOUT=100).
set -x
timeout 600 python -m pytest tests/test_gpu_api.py -m gpu -q -p no:cacheprovider -k "every_real_capable" 2>&1 | tail -2
for round in 1 2 3; do
  NS=2048 VARIANT_DOUBLE_2048=0 python tools/real_input_probe.py 2>&1 | grep double
  NS=2048 VARIANT_DOUBLE_2048=17 python tools/real_input_probe.py 2>&1 | grep double
  SFFT_SMEM_CARVEOUT=100 NS=2048 VARIANT_DOUBLE_2048=17 python tools/real_input_probe.py 2>&1 | grep double
done
