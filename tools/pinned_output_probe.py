import time, torch, numpy as np, sys
sys.path.insert(0,'.')
import paper_2203_09384_b200 as sf
B,N=65536,1024
X=sf.generate_batch(B,N,seed=1)
plan=sf.make_plan(N)
sf.execute(plan, X[:1024])
def t(fn):
    t0=time.perf_counter(); r=fn(); return time.perf_counter()-t0, r
dt,_=t(lambda: torch.empty((B,N),dtype=torch.complex64,pin_memory=True)); print('first pinned alloc 512MiB', dt*1e3)
dt,_=t(lambda: torch.empty((B,N),dtype=torch.complex64,pin_memory=True)); print('second (cached) pinned alloc', dt*1e3)
for i in range(3):
    dt,_=t(lambda: sf.execute(plan, X)); print('pageable execute', dt*1e3)
def pinned_out():
    o=torch.empty((B,N),dtype=torch.complex64,pin_memory=True).numpy()
    return sf.execute(plan, X, out=o)
for i in range(4):
    dt,_=t(pinned_out); print('pageable in, fresh pinned out (torch cache)', dt*1e3)
xp=torch.from_numpy(X).pin_memory().numpy()
for i in range(3):
    dt,_=t(lambda: sf.execute(plan, xp)); print('pinned in, fresh THP out', dt*1e3)
for s in (1<<20, 16<<20, 128<<20, 1<<30):
    dt,_=t(lambda: torch.empty(s,dtype=torch.uint8,pin_memory=True)); print('first pinned alloc', s>>20,'MiB', dt*1e3)
