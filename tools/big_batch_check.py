"""> 2^31 rows in one launch (fp32 N=2, 32 GiB in + 32 GiB out): sampled rows vs numpy, round trip (dev check)."""
import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2203_09384_b200 as sf
rows = (1 << 31) + 5
x = torch.empty((rows, 2), dtype=torch.complex64, device='cuda')
x.real.uniform_(-1, 1); x.imag.uniform_(-1, 1)
plan = sf.make_plan(2)
y = sf.execute(plan, x)
idx = torch.tensor([0, 1, (1 << 31) - 1, 1 << 31, rows - 1], device='cuda')
xs = x[idx].cpu().numpy().astype(np.complex128); ys = y[idx].cpu().numpy()
want = np.fft.fft(xs, axis=1)
print('rows', rows, 'max err', np.abs(ys - want).max())
z = sf.execute(sf.make_plan(2, 'inverse'), y)
print('roundtrip max', (z - x).abs().max().item())
