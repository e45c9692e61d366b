# fp32 real-input kernels: register cap (min-blocks) to keep the complex kernel's occupancy.
# Variant 0 vs the capped copy (N=512: 6, N=1024: 11, N=2048: 14), interleaved rounds, plus parity.
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -q -p no:cacheprovider -k "all_kernel_variants or every_real_capable or real" 2>&1 | tail -3
for round in 1 2 3; do
  NS=512 VARIANT_SINGLE_512=0 python tools/real_input_probe.py 2>&1 | grep single
  NS=512 VARIANT_SINGLE_512=6 python tools/real_input_probe.py 2>&1 | grep single
  NS=1024 VARIANT_SINGLE_1024=0 python tools/real_input_probe.py 2>&1 | grep single
  NS=1024 VARIANT_SINGLE_1024=11 python tools/real_input_probe.py 2>&1 | grep single
  NS=2048 VARIANT_SINGLE_2048=0 python tools/real_input_probe.py 2>&1 | grep single
  NS=2048 VARIANT_SINGLE_2048=14 python tools/real_input_probe.py 2>&1 | grep single
done
