"""Real-valued input rows: fused real loader (sfft_execute_ex, SFFT_INPUT_REAL)
vs widening to complex first and running the complex kernel (dev tool).
Batch = 1 GiB of complex output per launch; GB/s counts the algorithmic bytes
of each path (real path: 4/8 B in + 8/16 B out per element)."""
import json, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402


def timed(fn, iters=10, rounds=5):
    out = []
    for _ in range(rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / iters * 1e3)
    return statistics.median(out)


for prec in ("single", "double"):
    rdt, cdt = (torch.float32, torch.complex64) if prec == "single" else (torch.float64, torch.complex128)
    resz = 4 if prec == "single" else 8
    for n in [int(a) for a in os.environ.get("NS", "2,8,32,64,256,1024,2048").split(",")]:
        rows = (1 << 30) // (n * 2 * resz)
        xr = torch.rand((rows, n), dtype=rdt, device="cuda")
        y = torch.empty((rows, n), dtype=cdt, device="cuda")
        plan = sf.make_plan(n, precision=prec, variant=int(os.environ.get(f"VARIANT_{prec.upper()}_{n}", "0")))
        fused = lambda: sf.launch(plan, xr, y, rows)  # noqa: E731
        widen = lambda: sf.launch(plan, xr.to(cdt), y, rows)  # noqa: E731
        for f in (fused, widen):
            f()
        tf, tw = timed(fused), timed(widen)
        print(json.dumps({"prec": prec, "n": n, "variant": plan.variant, "rows": rows, "fused_us": round(tf, 1), "widen_then_c2c_us": round(tw, 1),
                          "speedup": round(tw / tf, 2),
                          "fused_gbs": round(rows * n * 3 * resz / tf / 1e3, 1)}), flush=True)
        del xr, y
        torch.cuda.empty_cache()
