# Host side of the multi-GPU e2e budget: CPU/NUMA layout, PCIe tree (all GPUs, even the ones
# this lease cannot use), host-memory copy bandwidth with 1..16 threads.
set -x
lscpu | grep -E "Model name|Socket|Core|Thread|NUMA|L3"
cat /proc/meminfo | head -3
nvidia-smi topo -m 2>&1 | head -20
lspci -tv 2>/dev/null | head -80
lspci 2>/dev/null | grep -ci nvidia
python - <<'PY'
import time, torch
n = 2 << 30
a = torch.empty(n, dtype=torch.uint8); b = torch.empty(n, dtype=torch.uint8)
a.fill_(1); b.fill_(2)
for t in (1, 2, 4, 8, 16):
    torch.set_num_threads(t)
    b.copy_(a)
    t0 = time.perf_counter()
    for _ in range(3):
        b.copy_(a)
    dt = (time.perf_counter() - t0) / 3
    print(f"host copy {t:2d} threads: {2 * n / dt / 1e9:.1f} GB/s (read+write)")
PY
