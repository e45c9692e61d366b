python tools/pcie_probe.py > gpurun_out/pcie.json 2>&1
for s in 2 3 4 6; do for c in 4 8 16 32 64; do SFFT_HOST_STREAMS=$s SFFT_HOST_CHUNK_MB=$c timeout 120 python tools/e2e_probe.py; done; done > gpurun_out/e2e_sweep.jsonl 2>&1
