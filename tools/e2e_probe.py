"""Time execute() on pinned host buffers (the bench e2e leg) for one host-pipeline shape.

    SFFT_HOST_SLOTS=4 SFFT_HOST_CHUNK_MB=16 python tools/e2e_probe.py [n] [batch]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
h_in = torch.empty((batch, n), dtype=torch.complex64, pin_memory=True)
h_out = torch.empty_like(h_in, pin_memory=True)
sf.generate_batch(batch, n, seed=0, out=h_in.numpy())
plan = sf.make_plan(n)
a, b = h_in.numpy(), h_out.numpy()
for _ in range(3):
    sf.execute(plan, a, out=b)
t = time.perf_counter()
reps = 10
for _ in range(reps):
    sf.execute(plan, a, out=b)
dt = (time.perf_counter() - t) / reps
print(json.dumps({"slots": os.environ.get("SFFT_HOST_SLOTS"), "chunk_mb": os.environ.get("SFFT_HOST_CHUNK_MB"),
                  "ms": round(dt * 1e3, 3), "gbs_each_way": round(batch * n * 8 / dt / 1e9, 1)}))
