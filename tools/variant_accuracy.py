"""Accuracy of every compiled kernel variant (twiddle-policy study).

For each precision, N and variant: max per-row rel-L2 vs the complex128
direct DFT over 256 Philox rows, and the ramp signal's max absolute
difference from the reference-formula direct DFT (the reference's own
tests/test_stats.py:211-222 bounds it by 0.1 at fp32 N = 2048).  One JSON
line per variant; argv[1] (optional) receives the list.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2203_09384_b200 as sf  # noqa: E402

lib = sf._native.lib()
out = []
for prec in ("single", "double"):
    for p in range(1, 12):
        n = 2**p
        x = sf.generate_batch(256, n, seed=p, precision=prec)
        exact = oracle.direct_dft(x)
        ramp = sf.generate("ramp", n, precision=prec)
        k = np.arange(n)
        ramp_exact = np.exp((-2.0j * np.pi / n) * (np.outer(k, k) % n)) @ ramp.astype(np.complex128)
        xd = torch.from_numpy(x).cuda()
        for v in range(lib.sfft_num_variants(n, 0 if prec == "single" else 1)):
            plan = sf.make_plan(n, precision=prec, variant=v)
            info = plan.kernel_info(0)
            y = sf.execute(plan, xd).cpu().numpy()
            yr = sf.execute(plan, ramp)
            rec = dict(prec=prec, n=n, variant=v, R=info["elems_per_thread"], twp=info["twiddle_policy"],
                       kernel=info["kernel"], loader=info["loader"],
                       rel_l2_max=float(np.max(np.linalg.norm(y - exact, axis=1) / np.linalg.norm(exact, axis=1))),
                       ramp_abs_max=float(np.abs(yr.astype(np.complex128) - ramp_exact).max()))
            out.append(rec)
            print(json.dumps(rec), flush=True)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
