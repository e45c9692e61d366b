"""Where does the host-buffer pipeline lose against the raw link? (dev tool)

Times, for 512 MiB in + 512 MiB out between pinned host buffers and HBM:
  a) one H2D and one D2H of the full size, concurrently, independent;
  b) the same bytes as 32 MiB chunks, H2D(k) -> D2H(k) dependency through an
     event, one stream per direction (no kernels);
  c) b) with a copy of the chunk on a third stream standing in for the kernel;
  d) execute(plan, pinned, out=pinned) -- the product path.
Each is timed back to back (calls may overlap) and synchronised per call.
Prints one JSON line of GB/s each way.
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

N, B = 1024, 65536
nbytes = N * B * 8
chunk = int(os.environ.get("CHUNK_MB", "32")) << 20
dev = torch.device("cuda:0")
h_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(nbytes, dtype=torch.uint8, device=dev)
d_out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
s_h2d, s_d2h, s_k = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, reps=5):
    """Back-to-back calls, one sync at the end (calls may overlap)."""
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def timed_sync(fn, reps=5):
    """Each call synchronised on its own (what one execute() costs)."""
    fn()
    torch.cuda.synchronize()
    best = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best.append(time.perf_counter() - t)
    return sorted(best)[len(best) // 2]


def full_concurrent():
    with torch.cuda.stream(s_h2d):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s_d2h):
        h_out.copy_(d_out, non_blocking=True)


def chunked(with_kernel):
    def run():
        for off in range(0, nbytes, chunk):
            sl = slice(off, min(nbytes, off + chunk))
            with torch.cuda.stream(s_h2d):
                d_in[sl].copy_(h_in[sl], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_h2d)
            src = d_in
            if with_kernel:
                s_k.wait_event(ev)
                with torch.cuda.stream(s_k):
                    d_out[sl].copy_(d_in[sl], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(s_k)
                src = d_out
            s_d2h.wait_event(ev)
            with torch.cuda.stream(s_d2h):
                h_out[sl].copy_(src[sl], non_blocking=True)
    return run


plan = sf.make_plan(N)
a = h_in.view(torch.complex64).view(B, N).numpy()
b = h_out.view(torch.complex64).view(B, N).numpy()
sf.generate_batch(B, N, seed=0, out=a)
res = {"chunk_mb": chunk >> 20}
for name, fn in (("a_full_concurrent", full_concurrent), ("b_chunked_copies", chunked(False)),
                 ("c_chunked_with_d2d", chunked(True)), ("d_execute", lambda: sf.execute(plan, a, out=b))):
    res[name] = round(nbytes / timed(fn) / 1e9, 1)
    res[name + "_synced"] = round(nbytes / timed_sync(fn) / 1e9, 1)
print(json.dumps(res))
