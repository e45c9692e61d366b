"""execute() on pinned numpy buffers: complex rows vs real rows (half the H2D
bytes through sfft_execute_host_ex), N=1024 x 65536 fp32 (dev tool)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

n, b = 1024, 65536
plan = sf.make_plan(n)
xc = torch.empty((b, n), dtype=torch.complex64, pin_memory=True).numpy()
xc[:] = sf.generate_batch(b, n, seed=0)
xr = torch.empty((b, n), dtype=torch.float32, pin_memory=True).numpy()
xr[:] = xc.real
out = torch.empty((b, n), dtype=torch.complex64, pin_memory=True).numpy()
res = {}
for name, x in (("complex_in", xc), ("real_in", xr)):
    for _ in range(2):
        sf.execute(plan, x, out=out)
    ts = []
    for _ in range(7):
        t = time.perf_counter()
        sf.execute(plan, x, out=out)
        ts.append(time.perf_counter() - t)
    res[name + "_ms"] = round(sorted(ts)[3] * 1e3, 2)
res["speedup"] = round(res["complex_in_ms"] / res["real_in_ms"], 2)
print(json.dumps(res))
