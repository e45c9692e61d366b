"""First-call cost of the host pipeline (dev tool): staging allocation, page faults."""
import time, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
t0 = time.perf_counter()
import torch
torch.cuda.init(); torch.empty(1, device="cuda")
print("cuda init", round((time.perf_counter() - t0) * 1e3, 1), "ms")
import paper_2203_09384_b200 as sf
B, N = 65536, 1024
X = sf.generate_batch(B, N, seed=1)
cudart = ctypes.CDLL("libcudart.so.12") if False else None
for label, fn in [
    ("plan create (first execute, 1 row)", lambda: sf.execute(sf.make_plan(N), X[:1])),
]:
    t = time.perf_counter(); fn(); print(label, round((time.perf_counter() - t) * 1e3, 1), "ms")
plan = sf.make_plan(N)
for i in range(3):
    t = time.perf_counter(); sf.execute(plan, X); print("execute 512 MiB pageable, call", i, round((time.perf_counter() - t) * 1e3, 1), "ms")
plan2 = sf.make_plan(N, "inverse")
t = time.perf_counter(); sf.execute(plan2, X); print("second plan, first large call", round((time.perf_counter() - t) * 1e3, 1), "ms")
t = time.perf_counter(); p = torch.empty(192 << 20, dtype=torch.uint8, pin_memory=True); print("pin 192 MiB", round((time.perf_counter() - t) * 1e3, 1), "ms")
import mmap
t = time.perf_counter()
m = mmap.mmap(-1, 512 << 20, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS); m.madvise(mmap.MADV_HUGEPAGE)
a = np.frombuffer(m, dtype=np.uint8); a[::4096] = 1
print("512 MiB THP mmap + first touch (1 thread)", round((time.perf_counter() - t) * 1e3, 1), "ms")
