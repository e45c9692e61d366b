"""Kernel time vs batch for one (N, precision): fits t = a + b*B to expose the fixed per-launch cost."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
prec = sys.argv[2] if len(sys.argv) > 2 else "single"
variants = [int(v) for v in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0"])]
esz = 8 if prec == "single" else 16
cdt = torch.complex64 if prec == "single" else torch.complex128
out = []
for v in variants:
    plan = sf.make_plan(n, precision=prec, variant=v)
    pts = []
    for b in (4096, 8192, 16384, 32768, 65536, 131072, 262144):
        rows = b * 1024 // n
        x = torch.empty((rows, n), dtype=cdt, device="cuda")
        x.real.uniform_(-1, 1)
        y = torch.empty_like(x)
        for _ in range(3):
            sf.launch(plan, x, y, rows)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        iters = 20
        for _ in range(iters):
            sf.launch(plan, x, y, rows)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / iters * 1e3
        pts.append((rows, us, 2 * rows * n * esz / us / 1e3))
        del x, y
    B = np.array([p[0] for p in pts], float)
    T = np.array([p[1] for p in pts])
    b1, a0 = np.polyfit(B, T, 1)
    rec = {"n": n, "prec": prec, "variant": v, "fixed_us": round(a0, 2),
           "asymptotic_gbs": round(2 * n * esz / b1 / 1e3, 1),
           "points": [(int(r), round(u, 2), round(g, 1)) for r, u, g in pts]}
    out.append(rec)
    print(json.dumps(rec), flush=True)
