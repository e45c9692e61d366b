"""Launch one kernel variant a few times on device-resident rows (ncu target).

    python tools/launch_variant.py N precision rows variant [launches]

REAL=1 feeds real rows (the SFFT_INPUT_REAL loader) instead of complex ones.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

n, prec, rows, variant = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
launches = int(sys.argv[5]) if len(sys.argv) > 5 else 5
dt = torch.complex64 if prec == "single" else torch.complex128
x = torch.randn((rows, n), dtype=dt, device="cuda")
y = torch.empty_like(x)
if os.environ.get("REAL") == "1":
    x = x.real.contiguous()
plan = sf.make_plan(n, precision=prec, variant=variant)
for _ in range(launches):
    sf.launch(plan, x, y, rows)
torch.cuda.synchronize()
print("variant", plan.variant, "ok")
