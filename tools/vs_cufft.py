"""The paper's comparison on B200: our kernels vs the vendor library (cuFFT).

    python tools/vs_cufft.py [--json out.json] [--bytes 1073741824]
    python tools/vs_cufft.py --latency [--json out.json]     # one transform per call

The paper benchmarks SYCL-FFT against cuFFT (PAPER.md:289-310, 380-386,
417-418).  This tool does the same for the B200 kernels: for every N and
precision it times, on the same 1 GiB device-resident batch, our default
kernel and cuFFT, interleaved round by round with CUDA events, and reports GB/s of algorithmic traffic for
both plus the accuracy of both against the complex128 direct DFT on 64 rows.
cuFFT is called two ways: directly (cufftPlanMany + cufftExecC2C/Z2Z through
ctypes, out-of-place into the same output buffer -- the library's own speed)
and through torch.fft.fft without `out=` (what a PyTorch user gets; with
`out=` torch adds a copy and halves the rate).  cuFFT is a measurement
reference only -- it is never on the product path.
"""
import argparse
import ctypes
import glob
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2203_09384_b200 as sf  # noqa: E402


def exact_dft(x):
    """O(N^2) forward DFT of every row in complex128 (no FFT rounding)."""
    x = np.asarray(x).astype(np.complex128)
    n = x.shape[-1]
    k = np.arange(n)
    return x @ np.exp(-2j * np.pi * np.outer(k, k) / n).T


def _cufft():
    import torch as _t
    cands = glob.glob(os.path.join(os.path.dirname(_t.__file__), "..", "nvidia", "cufft", "lib", "libcufft.so*"))
    cands += ["libcufft.so.11", "/usr/local/cuda/lib64/libcufft.so"]
    for c in cands:
        try:
            return ctypes.CDLL(c)
        except OSError:
            continue
    raise RuntimeError("libcufft not found")


class CufftPlan:
    """Batched 1-D out-of-place C2C (fp32) / Z2Z (fp64) plan on the current stream."""

    def __init__(self, n, rows, prec):
        self.lib = _cufft()
        self.h = ctypes.c_int(0)
        dims = (ctypes.c_int * 1)(n)
        typ = 0x29 if prec == "single" else 0x69  # CUFFT_C2C / CUFFT_Z2Z
        rc = self.lib.cufftPlanMany(ctypes.byref(self.h), 1, dims, None, 1, n, None, 1, n, typ, int(rows))
        if rc != 0:
            raise RuntimeError(f"cufftPlanMany failed: {rc}")
        self.lib.cufftSetStream(self.h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        self.exec = self.lib.cufftExecC2C if prec == "single" else self.lib.cufftExecZ2Z

    def __call__(self, x, y):
        rc = self.exec(self.h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), -1)  # CUFFT_FORWARD
        if rc != 0:
            raise RuntimeError(f"cufftExec failed: {rc}")

    def __del__(self):
        try:
            self.lib.cufftDestroy(self.h)
        except Exception:
            pass


def timed(fn, iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


def latency(args):
    """Paper Table 2 on B200: one transform per call, 1000 timed calls after a
    warm-up, host wall clock per call (launch + stream sync), mean and min
    ("optimal").  Both arms are driven from Python
    through ctypes, so the host overhead is the same kind on both sides."""
    import time

    out = []
    stream = torch.cuda.current_stream()
    for n in [2**p for p in range(3, 12)]:
        x = torch.empty((1, n), dtype=torch.complex64, device="cuda")
        x.real.uniform_(-1, 1)
        x.imag.uniform_(-1, 1)
        y = torch.empty_like(x)
        plan = sf.make_plan(n, "forward")
        cplan = CufftPlan(n, 1, "single")
        arms = {
            "ours_launch_sync": lambda: (sf.launch(plan, x, y, 1, stream=stream), stream.synchronize()),
            "cufft_exec_sync": lambda: (cplan(x, y), stream.synchronize()),
            "ours_execute": lambda: sf.execute(plan, x),
        }
        rec = {"n": n}
        for name, fn in arms.items():
            for _ in range(50):
                fn()
            ts = []
            for _ in range(args.latency_calls):
                t0 = time.perf_counter_ns()
                fn()
                ts.append((time.perf_counter_ns() - t0) / 1e3)
            rec[name + "_mean_us"] = round(statistics.mean(ts), 2)
            rec[name + "_min_us"] = round(min(ts), 2)
        del cplan
        out.append(rec)
        print(json.dumps(rec), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--latency", action="store_true", help="single-transform latency protocol instead")
    ap.add_argument("--latency-calls", type=int, default=1000)
    ap.add_argument("--bytes", type=int, default=1 << 30)
    ap.add_argument("--n", default=",".join(str(2**p) for p in range(1, 12)))
    ap.add_argument("--prec", default="single,double")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    if args.latency:
        out = latency(args)
        if args.json:
            with open(args.json, "w") as f:
                json.dump(out, f, indent=1)
        return
    out = []
    for prec in args.prec.split(","):
        esz = 8 if prec == "single" else 16
        cdt = torch.complex64 if prec == "single" else torch.complex128
        for n in map(int, args.n.split(",")):
            rows = args.bytes // (n * esz)
            x = torch.empty((rows, n), dtype=cdt, device="cuda")
            x.real.uniform_(-1, 1)
            x.imag.uniform_(-1, 1)
            y = torch.empty_like(x)
            plan = sf.make_plan(n, "forward", precision=prec)
            cplan = CufftPlan(n, rows, prec)
            ours = lambda: sf.launch(plan, x, y, rows)  # noqa: E731
            lib = lambda: cplan(x, y)  # noqa: E731
            tfft = lambda: torch.fft.fft(x, dim=-1)  # noqa: E731
            for f in (ours, lib, tfft, ours, lib, tfft):
                f()
            t_ours, t_lib, t_torch = [], [], []
            for _ in range(args.rounds):
                t_ours.append(timed(ours, args.iters))
                t_lib.append(timed(lib, args.iters))
                t_torch.append(timed(tfft, args.iters))
            us_o, us_l, us_t = statistics.median(t_ours), statistics.median(t_lib), statistics.median(t_torch)
            del cplan
            gbs = lambda us: 2 * rows * n * esz / us / 1e3  # noqa: E731
            # accuracy on a 64-row sample against the exact (complex128) DFT
            xs = x[:64].cpu().numpy()
            exact = exact_dft(xs)
            sf.launch(plan, x[:64].contiguous(), y[:64], 64)
            e_o = np.max(np.linalg.norm(y[:64].cpu().numpy() - exact, axis=1) / np.linalg.norm(exact, axis=1))
            e_l = np.max(np.linalg.norm(torch.fft.fft(x[:64], dim=-1).cpu().numpy() - exact, axis=1)
                         / np.linalg.norm(exact, axis=1))
            rec = {"prec": prec, "n": n, "rows": rows, "ours_us": round(us_o, 2), "cufft_us": round(us_l, 2),
                   "torch_fft_us": round(us_t, 2),
                   "ours_gbs": round(gbs(us_o), 1), "cufft_gbs": round(gbs(us_l), 1),
                   "torch_fft_gbs": round(gbs(us_t), 1),
                   "speedup_vs_cufft": round(us_l / us_o, 3),
                   "ours_rel_l2_vs_exact": float(e_o), "cufft_rel_l2_vs_exact": float(e_l)}
            out.append(rec)
            print(json.dumps(rec), flush=True)
            del x, y
            torch.cuda.empty_cache()
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
