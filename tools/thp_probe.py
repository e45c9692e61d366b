"""Fresh-output allocation for execute() on pageable numpy (dev tool): np.empty
vs an anonymous mmap with MADV_HUGEPAGE, N=1024 x 65536 fp32."""
import json, mmap, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09384_b200 as sf  # noqa: E402

n, b = 1024, 65536
plan = sf.make_plan(n)
x = sf.generate_batch(b, n, seed=0)


def thp_empty(shape, dtype):
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(m, dtype=dtype).reshape(shape)


res = {}
for name, alloc in (("np_empty", lambda: np.empty(x.shape, np.complex64)), ("mmap_thp", lambda: thp_empty(x.shape, np.complex64))):
    ts = []
    for _ in range(6):
        t = time.perf_counter()
        out = alloc()
        sf.execute(plan, x, out=out)
        ts.append(time.perf_counter() - t)
        del out
    res[name] = round(sorted(ts)[len(ts) // 2] * 1e3, 2)
print(json.dumps(res))
