import time, ctypes, torch, statistics
import sys; sys.path.insert(0, '.')
import paper_2203_09384_b200 as sf
from paper_2203_09384_b200 import _native
x = torch.randn(1, 1024, dtype=torch.complex64, device='cuda')
y = torch.empty_like(x)
plan = sf.make_plan(1024)
sf.execute(plan, x)
st = torch.cuda.current_stream()
h = plan.native_handle(0)
lib = _native.lib()
def T(name, fn, n=3000):
    for _ in range(200): fn()
    ts=[]
    for _ in range(n):
        t=time.perf_counter_ns(); fn(); ts.append(time.perf_counter_ns()-t)
    ts.sort(); print(f"{name:40s} median {ts[len(ts)//2]/1e3:7.2f} us  min {ts[0]/1e3:7.2f}")
T("torch.empty_like", lambda: torch.empty_like(x))
T("torch.cuda.current_stream", lambda: torch.cuda.current_stream(x.device))
T("plan.native_handle", lambda: plan.native_handle(0))
T("x.to(c64).contiguous()", lambda: x.to(torch.complex64).contiguous())
T("data_ptr x2 + c_void_p", lambda: (ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())))
a, b, s = ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(st.cuda_stream)
T("sfft_execute (async launch only)", lambda: lib.sfft_execute(h, a, b, 1, s, None))
torch.cuda.synchronize()
T("sfft_execute_sync (launch+sync+flag)", lambda: lib.sfft_execute_sync(h, a, b, 1, s, None))
T("stream.synchronize (idle)", lambda: st.synchronize())
T("sf.launch + sync", lambda: (sf.launch(plan, x, y, 1, stream=st), st.synchronize()))
T("sf.execute", lambda: sf.execute(plan, x))
T("sf.execute out=y", lambda: sf.execute(plan, x, out=y))
