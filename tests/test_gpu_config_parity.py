"""Parity at the exact BASELINE.json config shapes, against the CPU oracle.

SURVEY.md 8(d) / VERDICT r1 "what's missing" 2: every config that the bench
measures is also checked row-for-row against the reference algorithm
(``oracle.reference_execute``, the bit-exact restatement of the reference's
``execute`` / ``FourierTransformer``, executor.py:50-96, estimator.py:61-68):

* configs[0]: fp32 forward N=8, B=4 (seed 0) plus 4 ramp rows -- every row vs
  the oracle and the exact DFT, tolerance 3e-5;
* configs[1]: fp32 forward N=1024, B=65536 -- ALL rows of the Philox batch
  (seed 1) vs the oracle;
* configs[2]: N=2..2048 x {fp32, fp64} x {forward, inverse} on the full 1 GiB
  batch; >= 4096 sampled rows (first, last, every CTA boundary of a 64-way
  split, random) carry the Philox rows of ``generate_batch(B, N, seed)``
  (reproduced row by row with ``oracle.generate_rows``) and are compared with
  the oracle; the other rows are filler -- each row's result depends only on
  its own input (bit-exact batch-position independence,
  test_gpu_parity.py::test_row_independent_of_batch_position);
* configs[3]: fp64 forward N=2048, B=131072 (4 GiB in), sampled the same way;
* configs[4]: fp32 forward N=512, B=262144 per GPU, sampled the same way.

Tolerances: the north star's, rel-L2 per row <= 1e-5*log2 N (fp32) /
1e-13*log2 N (fp64), against the oracle AND (on a 256-row subset) the exact
complex128 DFT.
"""

import numpy as np
import pytest

import oracle
import paper_2203_09384_b200 as sf
from conftest import row_rel_l2, tolerance

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GIB = 1 << 30


def dtype_of(prec):
    return np.complex64 if prec == "single" else np.complex128


def sample_rows(rows: int, per_cta: int, seed: int, count: int = 4096) -> np.ndarray:
    """First, last, rows around 64 evenly spaced CTA boundaries, and random rows."""
    picked = {0, 1, rows - 2, rows - 1}
    for k in range(1, 64):
        b = (k * rows // 64) // per_cta * per_cta
        picked.update({max(0, b - 1), b, min(rows - 1, b + 1)})
    rng = np.random.default_rng(seed)
    rnd = rng.choice(rows, size=min(count, rows), replace=False)
    return np.unique(np.concatenate([np.fromiter(picked, np.int64), rnd]))


def check_sampled(n, prec, direction, rows, seed, cuda, count=4096):
    """Full-size batch whose sampled rows are the Philox rows; compare them."""
    dt = dtype_of(prec)
    cdt = torch.complex64 if prec == "single" else torch.complex128
    plan = sf.make_plan(n, direction, precision=prec)
    idx = sample_rows(rows, plan.kernel_info(cuda.index or 0)["seqs_per_cta"], seed, count)
    xs = oracle.generate_rows(rows, n, idx, seed, dt)
    x = torch.empty((rows, n), dtype=cdt, device=cuda)
    torch.view_as_real(x).uniform_(-1.0, 1.0)
    tidx = torch.from_numpy(idx).to(cuda)
    x[tidx] = torch.from_numpy(xs).to(cuda)
    y = sf.execute(plan, x)
    got = y[tidx].cpu().numpy()
    del x, y
    torch.cuda.empty_cache()
    tol = tolerance(n, prec)
    want = oracle.reference_execute(xs, direction, dtype=dt)
    assert len(idx) >= min(count, rows)
    assert row_rel_l2(got, want).max() <= tol
    sub = slice(0, 256)
    assert row_rel_l2(got[sub], oracle.direct_dft(xs[sub], direction)).max() <= tol


def test_config0_n8_batch4(cuda):
    x = np.concatenate([oracle.generate_batch(4, 8, 0), np.tile(oracle.generate("ramp", 8), (4, 1))])
    got = sf.execute(sf.make_plan(8), torch.from_numpy(x).to(cuda)).cpu().numpy()
    assert row_rel_l2(got, oracle.reference_execute(x, "forward")).max() <= 3e-5
    assert row_rel_l2(got, oracle.direct_dft(x)).max() <= 3e-5


def test_config1_all_rows(cuda):
    """configs[1] in full: all 65536 Philox rows vs the reference algorithm."""
    rows, n = 65536, 1024
    x = sf.generate_batch(rows, n, seed=1)
    y = sf.execute(sf.make_plan(n), torch.from_numpy(x).to(cuda)).cpu().numpy()
    want = oracle.reference_execute(x, "forward")
    err = row_rel_l2(y, want)
    assert err.shape == (rows,) and err.max() <= tolerance(n, "single")
    # host API on the same rows (sfft_execute_host pipeline): bit-identical
    assert np.array_equal(sf.execute(sf.make_plan(n), x), y)


@pytest.mark.parametrize("direction", ["forward", "inverse"])
@pytest.mark.parametrize("prec", ["single", "double"])
@pytest.mark.parametrize("n", [2**p for p in range(1, 12)])
def test_config2_sampled_rows(cuda, n, prec, direction):
    rows = GIB // (n * (8 if prec == "single" else 16))
    check_sampled(n, prec, direction, rows, seed=2, cuda=cuda)


def test_config3_fp64_2048_sampled_rows(cuda):
    check_sampled(2048, "double", "forward", 131072, seed=3, cuda=cuda)


def test_config4_fp32_512_sampled_rows(cuda):
    check_sampled(512, "single", "forward", 262144, seed=4, cuda=cuda)
