"""Small launches of every compiled kernel variant, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py --quick
    compute-sanitizer --tool synccheck python tools/sanitize_run.py --quick
    compute-sanitizer --tool racecheck python tools/sanitize_run.py --n 2048 --prec double  (every variant of one size)

Batches are odd-sized so partial CTAs / partial warp tiles are exercised.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

quick = "--quick" in sys.argv
# --loader L: only the variants with that input path (e.g. 2 = persistent TMA pipeline)
only_loader = int(sys.argv[sys.argv.index("--loader") + 1]) if "--loader" in sys.argv else None
only_n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else None
only_prec = sys.argv[sys.argv.index("--prec") + 1] if "--prec" in sys.argv else None
lib = sf._native.lib()
count = 0
for prec in ("single", "double"):
    if only_prec is not None and prec != only_prec:
        continue
    for p in range(1, 12):
        n = 2**p
        if only_n is not None and n != only_n:
            continue
        nvar = lib.sfft_num_variants(n, 0 if prec == "single" else 1)
        for v in range(1 if quick and only_loader is None else nvar):
            if only_loader is not None and sf._native.variant_info(n, 0 if prec == "single" else 1, v)["loader"] != only_loader:
                continue
            for d in ("forward", "inverse"):
                batch = 37 if quick else 261
                x = torch.from_numpy(sf.generate_batch(batch, n, seed=1, precision=prec)).cuda()
                plan = sf.make_plan(n, d, precision=prec, variant=v)
                y = sf.execute(plan, x)
                buf = x.clone()
                sf.launch(plan, buf, buf, batch)  # in-place
                torch.cuda.synchronize()
                assert torch.equal(buf, y)
                count += 1
                if plan.supports_real_input(0):  # real-input loader of the default kernels
                    xr = x.real.contiguous()
                    assert torch.equal(sf.execute(plan, xr), sf.execute(plan, xr.to(x.dtype)))
                    count += 1
print(f"sanitize_run: {count} launches OK")
