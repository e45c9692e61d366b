# Real-valued input: every variant with the default's arithmetic (same R, passes, twiddle policy;
# other SEQ / loader / layout) that has a real loader, two interleaved rounds.
set -x
timeout 600 python -m pytest tests/test_gpu_api.py -q -p no:cacheprovider -k "real" 2>&1 | tail -1
for rep in 1 2; do
  for v in 0 10 11 12; do VARIANT_SINGLE_2048=$v NS=2048 python tools/real_input_probe.py 2>&1 | grep '"single"'; done
  for v in 0 8 9; do VARIANT_DOUBLE_1024=$v NS=1024 python tools/real_input_probe.py 2>&1 | grep '"double"'; done
  for v in 0 4 15; do VARIANT_DOUBLE_2048=$v NS=2048 python tools/real_input_probe.py 2>&1 | grep '"double"'; done
done
