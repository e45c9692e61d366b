# Host pipeline: minimum chunk 2 MiB (default) vs 1 MiB / 512 KiB for 2-16 MiB calls
set -x
for r in 1 2 3; do
  for kb in 2048 1024 512; do SIZES_MIB=2,3,4,8,16 SFFT_HOST_MIN_CHUNK_KB=$kb timeout 300 python tools/e2e_size_probe.py; done
done
