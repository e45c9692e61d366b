"""Probe host<->device copy bandwidth (pinned), for the e2e roofline."""
import json
import time

import torch

n = 512 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
res = {}
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize(); res[name] = 5 * n / (time.perf_counter() - t) / 1e9
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); res["bidir_each"] = 5 * n / (time.perf_counter() - t) / 1e9
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
