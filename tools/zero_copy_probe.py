"""Host-buffer latency: zero-copy staging vs the copy-engine small-call path.

Run twice -- SFFT_ZERO_COPY_BYTES=0 (copies) and =1048576 (zero-copy up to
1 MiB) -- and compare.  execute(plan, numpy) median / min over 300 calls per
point, fp32 and fp64, one row and small batches; each output is checked
against the device path.  One JSON line per point.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

mode = os.environ.get("SFFT_ZERO_COPY_BYTES", "default")
for prec in ("single", "double"):
    for n, rows in ((8, 1), (64, 1), (256, 1), (1024, 1), (2048, 1), (1024, 4), (1024, 8), (2048, 8),
                    (1024, 32), (1024, 64), (2048, 32)):
        x = sf.generate_batch(rows, n, seed=3, precision=prec)
        if rows == 1:
            x = x[0]
        plan = sf.make_plan(n, precision=prec)
        ref = sf.execute(plan, torch.from_numpy(np.ascontiguousarray(x)).cuda()).cpu().numpy()
        y = sf.execute(plan, x)
        assert np.array_equal(y, ref), (prec, n, rows)
        ts = []
        for _ in range(300):
            t0 = time.perf_counter_ns()
            sf.execute(plan, x)
            ts.append((time.perf_counter_ns() - t0) / 1e3)
        ts.sort()
        print(json.dumps({"mode": mode, "prec": prec, "n": n, "rows": rows, "out_bytes": y.nbytes,
                          "median_us": round(ts[len(ts) // 2], 2), "min_us": round(ts[0], 2)}), flush=True)
