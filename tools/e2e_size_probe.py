"""Host-buffer execute() time vs call size, pinned and pageable (dev tool).

    SFFT_HOST_SPLIT=8 python tools/e2e_size_probe.py

fp32 N=1024 rows; sizes 2..512 MiB each way; median of 7 calls after 2 warm-ups.
Prints one JSON line per (size, memory kind): ms and GB/s each way.
"""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

n = 1024
plan = sf.make_plan(n)
for mib in [int(m) for m in os.environ.get("SIZES_MIB", "2,4,8,16,32,64,128,512").split(",")]:
    rows = (mib << 20) // (n * 8)
    for kind in ("pinned", "pageable"):
        if kind == "pinned":
            a = torch.empty((rows, n), dtype=torch.complex64, pin_memory=True).numpy()
            b = torch.empty((rows, n), dtype=torch.complex64, pin_memory=True).numpy()
        else:
            a = np.empty((rows, n), np.complex64)
            b = np.empty((rows, n), np.complex64)
        sf.generate_batch(rows, n, seed=1, out=a)
        for _ in range(2):
            sf.execute(plan, a, out=b)
        ts = []
        for _ in range(7):
            t = time.perf_counter()
            sf.execute(plan, a, out=b)
            ts.append(time.perf_counter() - t)
        dt = statistics.median(ts)
        print(json.dumps({"split": os.environ.get("SFFT_HOST_SPLIT", "default"), "min_chunk_kb": os.environ.get("SFFT_HOST_MIN_CHUNK_KB", "2048"), "mib": mib, "kind": kind,
                          "ms": round(dt * 1e3, 3), "gbs_each_way": round(rows * n * 8 / dt / 1e9, 1)}), flush=True)
