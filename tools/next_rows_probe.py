"""Measurement of the SURVEY 8(f) rows around the path (the callers either side).

* (f)2 batched FourierTransformer: ``fit_transform`` on BASELINE configs[1]
  (65536 x 1024 complex64, numpy in / numpy out -- the reference's calling
  convention) against the reference's per-row ``_apply`` loop
  (estimator.py:61-68) restated on the CPU (the oracle port called one row at
  a time), timed on a row sample;
* (f)3 verification: ``stats.verify_batch`` (per-row chi-square on the GPU)
  over all 65536 rows vs ``stats.compare_spectra`` (the reference's per-pair
  report, stats.py:209-239) per row on the host, timed on a sample;
* execute() with plain (pageable) numpy vs pinned host buffers, same batch.

Prints one JSON line per measurement.  Test/measurement infrastructure only:
the oracle is the CPU side of the comparison.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2203_09384_b200 as sf  # noqa: E402
from paper_2203_09384_b200.oracle import naive_dft_batch  # noqa: E402
from paper_2203_09384_b200.stats import compare_spectra, verify_batch  # noqa: E402

B, N = 65536, 1024
X = sf.generate_batch(B, N, seed=1)


def best(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return min(ts)


# (f)2 FourierTransformer
est = sf.FourierTransformer().fit(X)
t_gpu = best(lambda: est.transform(X))
sample = 2048
t0 = time.perf_counter()
ref = np.stack([oracle.reference_execute(row[None], "forward")[0] for row in X[:sample]])
t_ref = (time.perf_counter() - t0) * B / sample
print(json.dumps({"row": "(f)2 FourierTransformer.transform", "rows": B, "n": N,
                  "gpu_s": round(t_gpu, 4), "gpu_rows_per_s": round(B / t_gpu),
                  "reference_per_row_loop_s_extrapolated": round(t_ref, 2),
                  "reference_rows_per_s": round(B / t_ref), "speedup": round(t_ref / t_gpu, 1),
                  "note": "numpy in/out through the host pipeline; reference = oracle port one row per call, "
                          f"1 core, {sample}-row sample"}), flush=True)
y = est.transform(X)
assert np.max(np.linalg.norm(y[:sample] - ref, axis=1) / np.linalg.norm(ref, axis=1)) <= 1e-4

# (f)3 verification
yd = torch.from_numpy(y).cuda()
exact = naive_dft_batch(torch.from_numpy(X).cuda(), precision="double")
torch.cuda.synchronize()
t_dft = best(lambda: (naive_dft_batch(torch.from_numpy(X[:8192]).cuda(), precision="double"),
                      torch.cuda.synchronize()), reps=3) * B / 8192
t_ver = best(lambda: verify_batch(yd, exact), reps=3)
rep = verify_batch(yd, exact)
sample = 256
ex_h = exact[:sample].cpu().numpy()
t0 = time.perf_counter()
for i in range(sample):
    compare_spectra(y[i], ex_h[i].astype(np.complex64))
t_cpu = (time.perf_counter() - t0) * B / sample
print(json.dumps({"row": "(f)3 verify_batch (per-row chi-square on the GPU)", "rows": B, "n": N,
                  "gpu_s": round(t_ver, 4), "direct_dft_zgemm_s": round(t_dft, 4),
                  "reference_compare_spectra_per_row_s_extrapolated": round(t_cpu, 2),
                  "speedup": round(t_cpu / t_ver, 1), "p_value_min": rep.p_value_min,
                  "max_rel_l2": rep.max_rel_l2}), flush=True)

# execute(): pageable vs pinned host buffers
plan = sf.make_plan(N)
t_pageable = best(lambda: sf.execute(plan, X))
xp = torch.from_numpy(X).pin_memory().numpy()
out = torch.empty((B, N), dtype=torch.complex64, pin_memory=True).numpy()
t_pinned = best(lambda: sf.execute(plan, xp, out=out))
gflop = B * 5 * N * np.log2(N) / 1e9
print(json.dumps({"row": "execute() host buffers", "rows": B, "n": N,
                  "pageable_ms": round(t_pageable * 1e3, 2), "pageable_gflops": round(gflop / t_pageable, 1),
                  "pinned_ms": round(t_pinned * 1e3, 2), "pinned_gflops": round(gflop / t_pinned, 1)}), flush=True)
