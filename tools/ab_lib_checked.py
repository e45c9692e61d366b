"""A/B of two builds of libsfft on checked launches (NaN/Inf flag passed), same process.

    python tools/ab_lib_checked.py tools/ab_lib/libsfft_prev.so [rounds]
Times sfft_execute with a device flag for the default kernel of several
(N, precision) points, alternating the current library and the given one;
reports the median GB/s of each.  Dev tool (the previous build is not in git).
"""
import ctypes, json, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402
from paper_2203_09384_b200 import _native  # noqa: E402

other = ctypes.CDLL(os.path.abspath(sys.argv[1]))
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 5
libs = {"current": _native.lib(), "previous": other}
for lib in libs.values():
    lib.sfft_plan_create.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_int64, ctypes.c_int32]
    lib.sfft_execute.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                 ctypes.c_void_p]
for n, prec in ((2048, 1), (1024, 1), (512, 1), (2048, 0), (1024, 0)):
    esz = 8 if prec == 0 else 16
    rows = (1 << 30) // (n * esz)
    cdt = torch.complex64 if prec == 0 else torch.complex128
    x = torch.empty((rows, n), dtype=cdt, device="cuda")
    torch.view_as_real(x).uniform_(-1, 1)
    y = torch.empty_like(x)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    plans = {}
    for name, lib in libs.items():
        h = ctypes.c_void_p()
        assert lib.sfft_plan_create(ctypes.byref(h), n, prec, 0, 0, 0) == 0
        plans[name] = h
    st = torch.cuda.current_stream().cuda_stream
    res = {k: [] for k in libs}
    for _ in range(rounds):
        for name, lib in libs.items():
            for _ in range(3):
                lib.sfft_execute(plans[name], x.data_ptr(), y.data_ptr(), rows, st, flag.data_ptr())
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                lib.sfft_execute(plans[name], x.data_ptr(), y.data_ptr(), rows, st, flag.data_ptr())
            b.record()
            torch.cuda.synchronize()
            res[name].append(2 * rows * n * esz / (a.elapsed_time(b) / 20 * 1e-3) / 1e9)
    assert int(flag.item()) == 0
    print(json.dumps({"n": n, "prec": "single" if prec == 0 else "double",
                      **{k: round(statistics.median(v), 1) for k, v in res.items()}}), flush=True)
    del x, y
    torch.cuda.empty_cache()
