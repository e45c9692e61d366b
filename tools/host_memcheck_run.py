"""Host-pipeline calls of every size class for compute-sanitizer (dev tool):
zero-copy (<= 1 MiB), small, mid-size split chunks and long 32 MiB chunks, pinned and pageable,
complex and real input, growing and shrinking between calls (slot reallocation)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

n = 1024
plan = sf.make_plan(n)
for mib in (0.5, 3, 8, 24, 80, 6, 40):
    rows = int(mib * (1 << 20)) // (n * 8)
    x = sf.generate_batch(rows, n, seed=3)
    want = np.fft.fft(x.astype(np.complex128), axis=1)
    for pinned in (False, True):
        a = torch.from_numpy(x).pin_memory().numpy() if pinned else x
        y = sf.execute(plan, a)
        err = np.max(np.linalg.norm(y - want, axis=1) / np.linalg.norm(want, axis=1))
        assert err < 1e-5 * 10, (mib, pinned, err)
    yr = sf.execute(plan, x.real.copy())
    assert np.max(np.abs(yr - np.fft.fft(x.real.astype(np.float64), axis=1))) < 1e-2
print("host_memcheck_run: OK")
