"""Sustained-load A/B of kernel variants (power/clock steady state).

    python tools/sustained.py N precision rows v0,v1,... [--secs 4] [--rounds 2]

Variant "copy" is torch's copy_ between the same buffers (read + write of the
same bytes, no FFT): the memory system's own sustained rate.

Each variant runs back to back for --secs seconds per round (variants
interleaved across rounds, so box drift hits all of them); blocks of 50
launches are timed with CUDA events and the GB/s of the second half of each
window (after the clocks have settled under the power cap) is kept.  NVML
samples SM clock and power during every window.  Prints one JSON line.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402


class Sampler:
    def __init__(self, index=0, period=0.05):
        self.samples, self.period, self.stop_flag = [], period, threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(index)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None

    def __enter__(self):
        self.samples.clear()
        self.stop_flag.clear()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def _run(self):
        while not self.stop_flag.is_set() and self.nv is not None:
            try:
                sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                pw = self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.samples.append((sm, pw))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self.stop_flag.set()
        self.t.join()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int)
    ap.add_argument("prec")
    ap.add_argument("rows", type=int)
    ap.add_argument("variants")
    ap.add_argument("--secs", type=float, default=4.0)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--direction", default="forward")
    a = ap.parse_args()
    esz = 8 if a.prec == "single" else 16
    cdt = torch.complex64 if a.prec == "single" else torch.complex128
    x = torch.empty((a.rows, a.n), dtype=cdt, device="cuda")
    x.real.uniform_(-1, 1)
    x.imag.uniform_(-1, 1)
    y = torch.empty_like(x)
    variants = [-1 if v == "copy" else int(v) for v in a.variants.split(",")]
    # variant -1: torch copy_ of the same buffers (the HBM reference stream)
    plans = {v: sf.make_plan(a.n, a.direction, precision=a.prec, variant=v) for v in variants if v >= 0}
    res = {v: [] for v in variants}
    clk = {v: [] for v in variants}
    pwr = {v: [] for v in variants}
    block = 50
    for _ in range(a.rounds):
        for v in variants:
            gbs = []
            with Sampler() as smp:
                t0 = time.time()
                while time.time() - t0 < a.secs:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(block):
                        if v < 0:
                            y.copy_(x)
                        else:
                            sf.launch(plans[v], x, y, a.rows)
                    e1.record()
                    e1.synchronize()
                    gbs.append(2 * a.rows * a.n * esz * block / (e0.elapsed_time(e1) * 1e-3) / 1e9)
            half = gbs[len(gbs) // 2:]
            res[v].append(statistics.median(half))
            tail = smp.samples[len(smp.samples) // 2:]
            if tail:
                clk[v].append(statistics.median(s[0] for s in tail))
                pwr[v].append(statistics.median(s[1] for s in tail))
    print(json.dumps({
        "n": a.n, "prec": a.prec, "dir": a.direction, "rows": a.rows, "secs": a.secs, "rounds": a.rounds,
        "steady_gbs": {v: round(statistics.median(g), 1) for v, g in res.items()},
        "per_round_gbs": {v: [round(t, 1) for t in g] for v, g in res.items()},
        "sm_mhz": {v: (round(statistics.median(c)) if c else None) for v, c in clk.items()},
        "power_w": {v: (round(statistics.median(p), 1) if p else None) for v, p in pwr.items()},
    }))


if __name__ == "__main__":
    main()
