"""Where the host-buffer latency of one small execute() goes (fp32 N=1024,
one row, pageable numpy): the Python layer vs the native call vs its parts.
Medians over 2000 calls."""
import ctypes
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402
from paper_2203_09384_b200 import _native  # noqa: E402


def med(fn, k=2000):
    ts = []
    for _ in range(k):
        t0 = time.perf_counter_ns()
        fn()
        ts.append((time.perf_counter_ns() - t0) / 1e3)
    return statistics.median(ts), min(ts)


for n in (8, 1024):
    plan = sf.make_plan(n)
    x = sf.generate_batch(1, n, seed=1)[0]
    out = np.empty_like(x)
    h = plan.native_handle(0)
    lib = _native.lib()
    xp = x.ctypes.data
    op = out.ctypes.data
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    st = torch.cuda.current_stream().cuda_stream
    rows = [
        ("sf.execute(plan, x)", lambda: sf.execute(plan, x)),
        ("sf.execute(plan, x, out=out)", lambda: sf.execute(plan, x, out=out)),
        ("sfft_execute_host (native only)", lambda: lib.sfft_execute_host(h, xp, op, 1)),
        ("sfft_execute + cudaStreamSynchronize", lambda: (lib.sfft_execute(h, xd.data_ptr(), yd.data_ptr(), 1, st, None),
                                                        torch.cuda.current_stream().synchronize())),
        ("cudaStreamSynchronize (idle)", lambda: torch.cuda.current_stream().synchronize()),
    ]
    for name, fn in rows:
        fn()
        m, lo = med(fn)
        print(f"N={n:5d} {name:40s} median {m:7.2f} us  min {lo:7.2f}")
