"""Cost of pinning pageable numpy buffers in place (cudaHostRegister) vs the
staged pageable path, 512 MiB (dev tool)."""
import json
import time

import numpy as np
import torch

cudart = torch.cuda.cudart()
torch.cuda.init()
res = {}
for mb in (32, 128, 512):
    a = np.ones(mb << 18, dtype=np.complex64)  # mb MiB
    ts_r, ts_u = [], []
    for _ in range(3):
        t = time.perf_counter()
        rc = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        ts_r.append(time.perf_counter() - t)
        t = time.perf_counter()
        cudart.cudaHostUnregister(a.ctypes.data)
        ts_u.append(time.perf_counter() - t)
    res[f"{mb}MiB_register_ms"] = round(min(ts_r) * 1e3, 2)
    res[f"{mb}MiB_unregister_ms"] = round(min(ts_u) * 1e3, 2)
print(json.dumps(res))
