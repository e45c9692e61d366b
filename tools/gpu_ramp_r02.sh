# Host pipeline chunk schedule: flat 32 MiB chunks vs ramped ends (SFFT_HOST_RAMP=R: first/last R chunks
# 1/2^R .. 1/2 of a full chunk), pinned e2e leg of bench (configs[1]), interleaved rounds; correctness
# of the host-path GPU tests under the ramp.
set -x
SFFT_HOST_RAMP=3 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
for round in 1 2 3 4; do
  for r in 0 2 3 4 5; do SFFT_HOST_RAMP=$r timeout 120 python tools/e2e_probe.py 1024 65536 | sed "s/^/ramp=$r /"; done
done
for r in 0 3 4; do SFFT_HOST_RAMP=$r timeout 120 python tools/e2e_probe.py 2048 32768 | sed "s/^/n2048 ramp=$r /"; done
