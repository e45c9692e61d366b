"""execute() on pageable vs pinned numpy buffers (host path), N=1024 x 65536."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

n, b = 1024, 65536
plan = sf.make_plan(n)
x = sf.generate_batch(b, n, seed=0)
out = np.empty_like(x)
res = {}
for name, (xi, xo) in {
    "pageable_in_fresh_out": (x, None),
    "pageable_in_pageable_out": (x, out),
    "pinned_in_pinned_out": (torch.from_numpy(x).pin_memory().numpy(), torch.empty((b, n), dtype=torch.complex64, pin_memory=True).numpy()),
}.items():
    for _ in range(2):
        sf.execute(plan, xi, out=xo)
    t = time.perf_counter()
    for _ in range(5):
        sf.execute(plan, xi, out=xo)
    res[name] = round((time.perf_counter() - t) / 5 * 1e3, 2)
print(json.dumps(res))
