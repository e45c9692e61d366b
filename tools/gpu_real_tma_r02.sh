# fp32 real input at N=512 / 1024: the default LDG real loader vs a bulk-TMA real loader on the same
# passes (variants 6 / 11; bit-identical by construction -- the loader does no arithmetic).
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -q -p no:cacheprovider -k "all_kernel_variants or every_real_capable or real" 2>&1 | tail -2
for round in 1 2 3; do
  NS=512 VARIANT_SINGLE_512=0 python tools/real_input_probe.py 2>&1 | grep single
  NS=512 VARIANT_SINGLE_512=6 python tools/real_input_probe.py 2>&1 | grep single
  NS=1024 VARIANT_SINGLE_1024=0 python tools/real_input_probe.py 2>&1 | grep single
  NS=1024 VARIANT_SINGLE_1024=11 python tools/real_input_probe.py 2>&1 | grep single
done
