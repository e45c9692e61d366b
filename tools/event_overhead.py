import torch, sys
sys.path.insert(0,'.')
import paper_2203_09384_b200 as sf
x = torch.randn(65536, 1024, dtype=torch.complex64, device='cuda'); y = torch.empty_like(x)
flag = torch.zeros(1, dtype=torch.int32, device='cuda')
plan = sf.make_plan(1024); st = torch.cuda.current_stream()
for _ in range(20): sf.launch(plan, x, y, 65536, stream=st, flag=flag)
K=50
for rep in range(4):
    a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(st)
    for _ in range(K): sf.launch(plan, x, y, 65536, stream=st, flag=flag)
    b.record(st); torch.cuda.synchronize(); plain = a.elapsed_time(b)/K
    evs=[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize(); a.record(st)
    for k in range(K):
        evs[k][0].record(st); sf.launch(plan, x, y, 65536, stream=st, flag=flag); evs[k][1].record(st)
    b.record(st); torch.cuda.synchronize(); withev = a.elapsed_time(b)/K
    kern = sum(e0.elapsed_time(e1) for e0,e1 in evs)/K
    print(f"plain {plain*1e3:.1f} us/step  with-events {withev*1e3:.1f} us/step  kernel {kern*1e3:.1f} us")
