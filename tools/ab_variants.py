"""Interleaved A/B timing of kernel variants (robust to box drift).

    python tools/ab_variants.py N precision rows v0,v1,... [rounds]
Each round times every variant for 20 launches in turn; reports the median
GB/s per variant over the rounds.
"""
import json, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

n, prec, rows = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
variants = [int(v) for v in sys.argv[4].split(",")]
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 7
ITERS = 50
esz = 8 if prec == "single" else 16
cdt = torch.complex64 if prec == "single" else torch.complex128
x = torch.empty((rows, n), dtype=cdt, device="cuda")
x.real.uniform_(-1, 1)
x.imag.uniform_(-1, 1)
y = torch.empty_like(x)
plans = {v: sf.make_plan(n, precision=prec, variant=v) for v in variants}
res = {v: [] for v in variants}
# clock spin-up: keep the GPU busy ~0.5 s so SM clocks leave their idle state
for v in variants:
    for _ in range(3):
        sf.launch(plans[v], x, y, rows)
t_spin = torch.cuda.Event(enable_timing=True)
t_end = torch.cuda.Event(enable_timing=True)
t_spin.record()
spins = 0
while True:
    for _ in range(20):
        sf.launch(plans[variants[0]], x, y, rows)
    spins += 20
    t_end.record()
    torch.cuda.synchronize()
    if t_spin.elapsed_time(t_end) > 500:
        break
for _ in range(rounds):
    for v in variants:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(ITERS):
            sf.launch(plans[v], x, y, rows)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / ITERS * 1e3
        res[v].append(2 * rows * n * esz / us / 1e3)
print(json.dumps({"n": n, "prec": prec, "rows": rows,
                  "median_gbs": {v: round(statistics.median(g), 1) for v, g in res.items()},
                  "spread": {v: round(max(g) - min(g), 1) for v, g in res.items()}}))
