"""BASELINE configs[2] at full size on the GPU: every N = 2^1..2^11, fp32 and
fp64, on a 1 GiB batch, checked through
size-independent properties plus a sampled exact comparison:

* forward then inverse returns the input (every row, checked on the device);
* Parseval over the whole batch (sum |X|^2 = N sum |x|^2, float64 sums);
* >= 4096 sampled rows -- first, last, CTA / warp-tile boundaries and random
  rows -- against numpy's complex128 FFT, per-row rel-L2 within tolerance.
"""

import numpy as np
import pytest

import paper_2203_09384_b200 as sf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GIB = 1 << 30


def row_rel(a, b):
    return (torch.linalg.vector_norm(a - b, dim=1) / torch.linalg.vector_norm(b, dim=1)).max().item()


@pytest.mark.parametrize("prec", ["single", "double"])
@pytest.mark.parametrize("n", [2**p for p in range(1, 12)])
def test_config3_full_batch(cuda, n, prec):
    esz = 8 if prec == "single" else 16
    rows = GIB // (n * esz)
    cdt = torch.complex64 if prec == "single" else torch.complex128
    g = torch.Generator(device=cuda).manual_seed(n)
    x = torch.empty((rows, n), dtype=cdt, device=cuda)
    x.real.uniform_(-1, 1, generator=g)
    x.imag.uniform_(-1, 1, generator=g)
    fwd = sf.make_plan(n, "forward", precision=prec)
    inv = sf.make_plan(n, "inverse", precision=prec)
    y = sf.execute(fwd, x)
    tol = (1e-5 if prec == "single" else 1e-13) * np.log2(n)

    # Parseval on the whole batch, float64 accumulation
    ex = x.abs().double().pow(2).sum().item()
    ey = y.abs().double().pow(2).sum().item()
    assert abs(ey / (n * ex) - 1.0) <= tol

    # sampled rows against numpy complex128: ends, CTA / tile boundaries, random
    per_cta = fwd.kernel_info(cuda.index)["seqs_per_cta"]
    edges = {0, 1, rows - 2, rows - 1}
    for k in range(1, 64):
        b = (k * rows // 64) // per_cta * per_cta
        edges.update({max(0, b - 1), b, min(rows - 1, b + 1)})
    rnd = torch.randperm(rows, generator=g, device=cuda)[:4096].cpu().numpy()  # distinct rows
    idx = np.unique(np.concatenate([np.array(sorted(edges)), rnd]))
    xs = x[torch.from_numpy(idx).to(cuda)].cpu().numpy().astype(np.complex128)
    want = np.fft.fft(xs, axis=1)
    got = y[torch.from_numpy(idx).to(cuda)].cpu().numpy().astype(np.complex128)
    err = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
    assert len(idx) >= 4096 and err.max() <= tol

    # round trip, every row, on the device
    z = sf.execute(inv, y)
    del y
    assert row_rel(z, x) <= 2 * tol
