"""Many small batched transforms: eager launches vs one CUDA graph replay (dev tool).

    python tools/graph_probe.py

For each (N, precision, rows) a chain of K launches alternating two buffers
(x -> y -> x ...) is timed three ways on one stream: eager `launch` calls
(programmatic dependent launch on), the same chain captured once into a CUDA
graph and replayed, and -- as the bandwidth reference -- the kernel time of a
single launch.  Prints one JSON line per point: us per transform call.
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

K = 200


def timed(fn, reps=5):
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e3)
    return statistics.median(out)


s = torch.cuda.Stream()
for n, prec, rows in ((64, "single", 16), (1024, "single", 64), (1024, "single", 1024), (2048, "double", 64)):
    cdt = torch.complex64 if prec == "single" else torch.complex128
    x = torch.randn((rows, n), dtype=cdt, device="cuda")
    y = torch.empty_like(x)
    plan = sf.make_plan(n, precision=prec)
    with torch.cuda.stream(s):
        def chain():
            for i in range(K):
                a, b = (x, y) if i % 2 == 0 else (y, x)
                sf.launch(plan, a, b, rows)
        chain()
        eager = timed(chain)
        g = torch.cuda.CUDAGraph()
        chain()  # warm
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            chain()
        replay = timed(g.replay)
        one = timed(lambda: sf.launch(plan, x, y, rows))
    print(json.dumps({"n": n, "prec": prec, "rows": rows, "calls": K,
                      "eager_us_per_call": round(eager / K, 2), "graph_us_per_call": round(replay / K, 2),
                      "single_launch_us": round(one, 2)}), flush=True)
