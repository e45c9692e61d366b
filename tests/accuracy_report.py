"""Accuracy table: GPU kernels vs the exact DFT, next to the reference engine's own error.

Report script (not a test module; lives in tests/ because it calls the
oracle).  For each N, precision and direction: 256 Philox rows; reports max per-row
rel-L2 of (a) the GPU result vs the complex128 direct DFT, (b) the reference
algorithm (oracle port, complex64 or complex128 stage engine) vs the same,
and (c) GPU vs reference.  Writes JSON to argv[1].
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # repo root
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2203_09384_b200 as sf  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    return float(np.max(np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)))


rows = []
for prec in ("single", "double"):
    dt = np.complex64 if prec == "single" else np.complex128
    for p in range(1, 12):
        n = 2**p
        x = sf.generate_batch(256, n, seed=p, precision=prec)
        exact = {d: oracle.direct_dft(x, d) for d in ("forward", "inverse")}
        for d in ("forward", "inverse"):
            gpu = sf.execute(sf.make_plan(n, d, precision=prec), torch.from_numpy(x).cuda()).cpu().numpy()
            ref = oracle.reference_execute(x, d, dtype=dt)
            rows.append({"precision": prec, "n": n, "direction": d, "gpu_vs_exact": rel(gpu, exact[d]),
                         "reference_vs_exact": rel(ref, exact[d]), "gpu_vs_reference": rel(gpu, ref),
                         "tolerance": (1e-5 if prec == "single" else 1e-13) * p})
            print(json.dumps(rows[-1]), flush=True)
with open(sys.argv[1] if len(sys.argv) > 1 else "accuracy.json", "w") as f:
    json.dump(rows, f, indent=1)
