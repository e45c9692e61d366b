"""Kernel sweep: every (precision, N, variant) on a fixed-size batch, CUDA events.

Development tool (not the bench contract): prints one line per config with the
kernel time and achieved algorithmic HBM GB/s (16*N B/row fp32, 32*N fp64).
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402


def time_plan(plan, x, y, rows, iters, warmup):
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        sf.launch(plan, x, y, rows, stream=stream)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    for _ in range(iters):
        sf.launch(plan, x, y, rows, stream=stream)
    stop.record(stream)
    torch.cuda.synchronize()
    return start.elapsed_time(stop) / iters * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=1 << 30, help="input buffer bytes")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--prec", default="single,double")
    ap.add_argument("--n", default=",".join(str(2**p) for p in range(1, 12)))
    ap.add_argument("--dir", default="forward")
    ap.add_argument("--all-variants", action="store_true")
    ap.add_argument("--variant", type=int, default=None)
    ap.add_argument("--json", default=None)
    ap.add_argument("--cool", type=float, default=0.0,
                    help="idle seconds before each timing (lets power/clocks recover)")
    args = ap.parse_args()
    peaks = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    peak = json.load(open(peaks))["hbm_gbs"] if os.path.exists(peaks) else 6549.8
    dev = torch.device("cuda:0")
    rows_out = []
    lib = sf._native.lib()
    for prec in args.prec.split(","):
        esz = 8 if prec == "single" else 16
        cdt = torch.complex64 if prec == "single" else torch.complex128
        for n in map(int, args.n.split(",")):
            rows = args.bytes // (n * esz)
            x = torch.empty((rows, n), dtype=cdt, device=dev)
            x.real.uniform_(-1, 1)
            x.imag.uniform_(-1, 1)
            y = torch.empty_like(x)
            nvar = lib.sfft_num_variants(n, 0 if prec == "single" else 1)
            vlist = range(nvar) if args.all_variants else [args.variant or 0]
            for v in vlist:
                plan = sf.make_plan(n, args.dir, precision=prec, variant=v)
                if args.cool > 0:
                    torch.cuda.synchronize()
                    time.sleep(args.cool)
                us = time_plan(plan, x, y, rows, args.iters, args.warmup)
                gbs = 2 * rows * n * esz / us / 1e3
                gflops = 5 * n * max(1, n.bit_length() - 1) * rows / us / 1e3
                info = plan.kernel_info(0)
                rec = dict(prec=prec, n=n, variant=v, rows=rows, us=round(us, 2), gbs=round(gbs, 1),
                           frac=round(gbs / peak, 3), gflops=round(gflops, 1),
                           kernel=info["kernel"], R=info["elems_per_thread"], seq=info["seqs_per_cta"],
                           threads=info["threads_per_cta"], radices=info["radices"])
                rows_out.append(rec)
                print(json.dumps(rec), flush=True)
            del x, y
            torch.cuda.empty_cache()
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rows_out, f, indent=1)


if __name__ == "__main__":
    main()
