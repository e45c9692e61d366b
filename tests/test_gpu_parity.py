"""GPU parity: the sm_100a kernels (through the C ABI) vs the CPU oracle.

Tolerances are the north star's: rel-L2 <= 1e-5*log2(N) in fp32 and
<= 1e-13*log2(N) in fp64, per row.  The oracle is the batched restatement of
the reference (oracle/stagefft_port.py), itself pinned bit-exactly to the
reference outputs in tests/golden (tests/test_oracle_golden.py).
"""

import numpy as np
import pytest

import oracle
import paper_2203_09384_b200 as sf
from conftest import rel_l2, row_rel_l2, tolerance

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ALL_N = [2**p for p in range(1, 12)]
PRECS = ["single", "double"]
DIRS = ["forward", "inverse"]


def dtype_of(prec):
    return np.complex64 if prec == "single" else np.complex128


def run(plan, x, dev):
    return sf.execute(plan, torch.from_numpy(np.ascontiguousarray(x)).to(dev)).cpu().numpy()


@pytest.mark.parametrize("direction", DIRS)
@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("n", ALL_N)
def test_all_lengths_vs_oracle(cuda, n, prec, direction):
    # odd batch: exercises partial CTAs / partial warp tiles
    batch = 1 + (3000 * 64) // n
    x = sf.generate_batch(batch, n, seed=n + (prec == "double"), precision=prec)
    plan = sf.make_plan(n, direction, precision=prec)
    got = run(plan, x, cuda)
    want = oracle.reference_execute(x, direction, dtype=dtype_of(prec))
    exact = oracle.direct_dft(x, direction)
    tol = tolerance(n, prec)
    assert row_rel_l2(got, want).max() <= tol
    assert row_rel_l2(got, exact).max() <= tol


@pytest.mark.parametrize("n", [2**p for p in range(3, 12)])
def test_golden_engine_fixtures(cuda, golden, n):
    """Reference `execute` outputs (complex64) for 4 signal kinds, both directions."""
    g = golden("engine_c64.npz")
    for kind in ("random", "ramp", "impulse", "constant"):
        x = g[f"in_{kind}_{n}"]
        for d in DIRS:
            got = run(sf.make_plan(n, d), x[None], cuda)[0]
            ref = g[f"out_{kind}_{n}_{d}"]
            assert rel_l2(got, ref) <= tolerance(n, "single"), (kind, d)


@pytest.mark.parametrize("n", [2, 4, 8, 16, 64])
def test_golden_split_radix_fixtures(cuda, golden, n):
    """N = 2, 4: the reference's split-radix route (kernels.py:205-232)."""
    g = golden("engine_c64.npz")
    x = g[f"in_split_{n}"]
    for d in DIRS:
        got = run(sf.make_plan(n, d, algorithm="split"), x[None], cuda)[0]
        assert rel_l2(got, g[f"out_split_{n}_{d}"]) <= tolerance(n, "single")


@pytest.mark.parametrize("n", ALL_N)
def test_golden_fp64_fixtures(cuda, golden, n):
    g = golden("restated_c128.npz")
    x = g[f"in_{n}"]
    for d in DIRS:
        got = run(sf.make_plan(n, d, precision="double"), x[None], cuda)[0]
        assert rel_l2(got, g[f"out_{n}_{d}"]) <= tolerance(n, "double")


def test_ramp8_closed_form(cuda):
    """RAMP8_SPECTRUM (reference tests/test_oracle.py:9-20)."""
    ramp8 = np.array([28, -4 + 9.65685424949238j, -4 + 4j, -4 + 1.6568542494923804j, -4,
                      -4 - 1.65685424949238j, -4 - 4j, -4 - 9.656854249492376j])
    for prec in PRECS:
        out = run(sf.make_plan(8, precision=prec), np.arange(8)[None].astype(dtype_of(prec)), cuda)[0]
        np.testing.assert_allclose(out, ramp8, atol=1e-5 if prec == "single" else 1e-12)


@pytest.mark.parametrize("prec", PRECS)
def test_impulse_and_constant(cuda, prec):
    for n in ALL_N:
        imp = np.zeros((3, n), dtype_of(prec))
        imp[:, 0] = 1
        np.testing.assert_allclose(run(sf.make_plan(n, precision=prec), imp, cuda), np.ones((3, n)), atol=1e-6)
        const = np.ones((2, n), dtype_of(prec))
        expect = np.zeros((2, n))
        expect[:, 0] = 1  # inverse of a constant is a unit impulse (test_executor.py:45-51)
        np.testing.assert_allclose(run(sf.make_plan(n, "inverse", precision=prec), const, cuda), expect, atol=1e-6)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("n", ALL_N)
def test_row_independent_of_batch_position(cuda, prec, n):
    """Determinism contract: a row's bits do not depend on batch size/position."""
    x = sf.generate_batch(517, n, seed=3, precision=prec)
    plan = sf.make_plan(n, precision=prec)
    full = run(plan, x, cuda)
    for i in (0, 1, 255, 516):
        assert np.array_equal(run(plan, x[i : i + 1], cuda)[0], full[i])
    assert np.array_equal(run(plan, x[100:300], cuda), full[100:300])
    assert np.array_equal(run(plan, x, cuda), full)  # repeat runs


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("n", [2, 16, 64, 1024, 2048])
def test_in_place(cuda, prec, n):
    x = torch.from_numpy(sf.generate_batch(300, n, seed=1, precision=prec)).to(cuda)
    plan = sf.make_plan(n, precision=prec)
    want = sf.execute(plan, x)
    buf = x.clone()
    sf.launch(plan, buf, buf, 300)
    torch.cuda.synchronize()
    assert torch.equal(buf, want)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("n", [2, 4, 8, 32, 128, 2048])
def test_nonfinite_input_raises(cuda, prec, n):
    plan = sf.make_plan(n, precision=prec)
    for row, col, val in ((0, 0, np.inf), (4, n - 1, np.nan), (1000, n // 2, -np.inf)):
        x = np.ones((1001, n), dtype_of(prec))
        x[row, col] = val
        with pytest.raises(sf.DomainError):
            sf.execute(plan, torch.from_numpy(x).to(cuda))
        with pytest.raises(sf.DomainError):
            sf.execute(plan, x)  # host path (sfft_execute_host)
    # imaginary part alone
    x = np.ones((7, n), dtype_of(prec))
    x[6, 0] = complex(0, np.nan)
    with pytest.raises(sf.DomainError):
        sf.execute(plan, x)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("n", [8, 256, 2048])
def test_host_path_matches_device_path(cuda, prec, n):
    # 40 MiB + a ragged tail: 2 chunks of the 32 MiB pipeline
    rows = (40 << 20) // (n * (8 if prec == "single" else 16)) + 3
    x = sf.generate_batch(rows, n, seed=5, precision=prec)
    plan = sf.make_plan(n, precision=prec)
    host = sf.execute(plan, x)
    dev = run(plan, x, cuda)
    assert isinstance(host, np.ndarray) and host.dtype == dtype_of(prec)
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("memory", ["pageable", "pinned", "pinned_in_pageable_out"])
def test_host_pipeline_reuses_slots(cuda, memory):
    """> 3 x 32 MiB so every device slot (and, for pageable memory, every
    pinned staging slot) is reused: exercises the per-slot event ordering of
    sfft_execute_host and the drain order of the staged path."""
    n, prec = 1024, "single"
    rows = (7 * (32 << 20) + (5 << 20)) // (n * 8) + 1  # 7.2 chunks, ragged tail
    x = sf.generate_batch(rows, n, seed=11, precision=prec)
    plan = sf.make_plan(n, precision=prec)
    want = run(plan, x[: rows // 3], cuda), run(plan, x[rows // 3:], cuda)
    if memory == "pageable":
        xin, out = x, np.empty_like(x)
    else:
        xin = torch.from_numpy(x).pin_memory().numpy()
        out = (torch.empty(x.shape, dtype=torch.complex64, pin_memory=True).numpy()
               if memory == "pinned" else np.empty_like(x))
    for _ in range(2):  # second call reuses the events of the first
        got = sf.execute(plan, xin, out=out)
        assert got is out
        assert np.array_equal(got[: rows // 3], want[0]) and np.array_equal(got[rows // 3:], want[1])
    # a NaN in the last chunk still raises, and the plan stays usable
    bad = x.copy()
    bad[-1, 5] = np.nan
    with pytest.raises(sf.DomainError):
        sf.execute(plan, bad)
    assert np.array_equal(sf.execute(plan, x)[:4], want[0][:4])


def test_input_dtypes_and_shapes(cuda):
    plan = sf.make_plan(8)
    # real float64 input is accepted (test_executor.py:89-92)
    out = sf.execute(plan, np.arange(8, dtype=np.float64))
    assert out.shape == (8,) and out.dtype == np.complex64
    assert rel_l2(out, oracle.direct_dft(np.arange(8))) <= 1e-4
    # integers, complex128 -> complex64 downcast (validation.py:26)
    assert np.array_equal(sf.execute(plan, np.arange(8)), out)
    assert np.array_equal(sf.execute(plan, np.arange(8).astype(np.complex128)), out)
    # torch CUDA real input stays on device and comes back complex64
    t = sf.execute(plan, torch.arange(8, dtype=torch.float32, device=cuda))
    assert t.is_cuda and t.dtype == torch.complex64
    assert np.array_equal(t.cpu().numpy(), out)
    with pytest.raises(sf.ShapeError):
        sf.execute(sf.make_plan(64), np.ones(32, np.complex64))
    with pytest.raises(sf.ShapeError):
        sf.execute(sf.make_plan(64), np.ones((2, 8, 8), np.complex64))
    with pytest.raises(sf.ShapeError):
        sf.execute(sf.make_plan(64), np.ones((8, 8), np.complex64))  # last axis != N
    with pytest.raises(sf.DomainError):
        sf.execute(plan, np.array(["a"] * 8))


def test_input_never_modified_output_fresh(cuda):
    plan = sf.make_plan(64)
    x = sf.generate_batch(10, 64, seed=9)
    snap = x.copy()
    a = sf.execute(plan, x)
    b = sf.execute(plan, x)
    assert np.array_equal(x, snap)
    assert not np.shares_memory(a, b) and not np.shares_memory(a, x)
    xt = torch.from_numpy(x).to(cuda)
    snapt = xt.clone()
    yt = sf.execute(plan, xt)
    assert torch.equal(xt, snapt) and yt.data_ptr() != xt.data_ptr()


def test_misaligned_view(cuda):
    base = torch.from_numpy(sf.generate_batch(1, 1 + 16 * 100, seed=2)).to(cuda).reshape(-1)
    view = base[1:].reshape(100, 16)  # 8-byte offset: not 16-byte aligned
    assert view.data_ptr() % 16 == 8
    plan = sf.make_plan(16)
    got = sf.execute(plan, view).cpu().numpy()
    assert np.array_equal(got, sf.execute(plan, view.cpu().numpy()))


@pytest.mark.parametrize(
    "n,prec,offset",
    [(2, "single", 1), (8, "single", 1), (8, "single", 3), (32, "single", 2), (2048, "single", 1),
     (8, "double", 1), (1024, "double", 1), (2048, "double", 1)],
)
def test_misaligned_real_view(cuda, n, prec, offset):
    """Real rows at a 4-byte (fp32) or 8-byte (fp64) offset: the tile, bulk-TMA
    and vectorised real loaders read 16-byte chunks.  execute() re-copies the
    view (bit-identical to an aligned copy); the raw entry points refuse it
    with SFFT_ERR_ARGUMENT instead of faulting -- and the context stays usable."""
    rdt = torch.float32 if prec == "single" else torch.float64
    rows = 37
    flat = torch.from_numpy(sf.generate_batch(1, offset + rows * n, seed=5, precision=prec).real.copy())
    flat = flat.to(rdt).to(cuda).reshape(-1)
    view = flat[offset:].reshape(rows, n)
    assert view.data_ptr() % 16 != 0
    plan = sf.make_plan(n, precision=prec)
    got = sf.execute(plan, view)
    aligned = view.clone()
    assert aligned.data_ptr() % 16 == 0
    want = sf.execute(plan, aligned)
    assert torch.equal(got, want)
    # widening to complex first gives the same bits (real loader == widening)
    assert torch.equal(got, sf.execute(plan, aligned.to(got.dtype)))
    out = torch.empty_like(want)
    with pytest.raises(sf.FftError, match="16-byte aligned"):
        sf.launch(plan, view, out, rows)
    lib = sf._native.lib()
    rc = lib.sfft_execute_ex(plan.native_handle(cuda.index or 0), view.data_ptr(), out.data_ptr(), rows,
                             None, None, sf._native.SFFT_INPUT_REAL)
    assert rc == 7  # SFFT_ERR_ARGUMENT
    torch.cuda.synchronize()
    assert torch.equal(sf.execute(plan, view), want)  # no sticky fault


@pytest.mark.parametrize("n,prec", [(8, "single"), (1024, "single"), (2048, "double")])
def test_overlapping_buffers(cuda, n, prec):
    """Input and output are disjoint or identical (complex in place).  Real
    rows under their own complex output, or a shifted complex view, would
    race between CTAs / pipeline chunks: every entry point refuses them with
    SFFT_ERR_ARGUMENT, and exact in-place stays bit-identical to out of place."""
    rows = 33
    cdt = torch.complex64 if prec == "single" else torch.complex128
    plan = sf.make_plan(n, precision=prec)
    x = torch.from_numpy(sf.generate_batch(rows + 1, n, seed=9, precision=prec)).to(cuda)
    want = sf.execute(plan, x[:rows])
    # exact in place
    buf = x[:rows].clone()
    sf.launch(plan, buf, buf, rows)
    torch.cuda.synchronize()
    assert torch.equal(buf, want)
    # shifted complex view: output one row after the input
    with pytest.raises(sf.FftError, match="overlap"):
        sf.launch(plan, x[:rows], x[1:], rows)
    # real rows inside their complex output buffer (same start address)
    out = torch.zeros((rows, n), dtype=cdt, device=cuda)
    real_view = out.view(torch.float32 if prec == "single" else torch.float64).reshape(-1)[: rows * n].reshape(rows, n)
    assert real_view.data_ptr() == out.data_ptr()
    with pytest.raises(sf.FftError, match="overlap"):
        sf.launch(plan, real_view, out, rows)
    with pytest.raises(sf.FftError, match="overlap"):
        sf.execute(plan, real_view, out=out)
    # the host pipeline: a real numpy view of the complex output array
    hout = np.zeros((rows, n), dtype=dtype_of(prec))
    hreal = hout.view(np.float32 if prec == "single" else np.float64).reshape(-1)[: rows * n].reshape(rows, n)
    with pytest.raises(sf.FftError, match="overlap"):
        sf.execute(plan, hreal, out=hout)
    torch.cuda.synchronize()
    assert torch.equal(sf.execute(plan, x[:rows]), want)  # context still usable


def test_shared_plan_across_threads(cuda):
    from concurrent.futures import ThreadPoolExecutor

    plan = sf.make_plan(256)
    signals = [sf.generate("random", 256, seed=s) for s in range(16)]
    expected = [sf.execute(plan, x) for x in signals]
    with ThreadPoolExecutor(max_workers=8) as pool:
        results = list(pool.map(lambda x: sf.execute(plan, x), signals))
    for got, want in zip(results, expected):
        assert np.array_equal(got, want)


@pytest.mark.parametrize("prec", PRECS)
def test_all_kernel_variants(cuda, prec):
    """Every compiled variant (the tuning space) is correct, not just the
    default -- forward and inverse against the exact DFT."""
    lib = sf._native.lib()
    for n in ALL_N:
        nvar = lib.sfft_num_variants(n, 0 if prec == "single" else 1)
        x = sf.generate_batch(333, n, seed=11, precision=prec)
        for direction in DIRS:
            want = oracle.direct_dft(x, direction)
            for v in range(nvar):
                got = run(sf.make_plan(n, direction, precision=prec, variant=v), x, cuda)
                assert row_rel_l2(got, want).max() <= tolerance(n, prec), (n, v, direction)


@pytest.mark.parametrize("direction", DIRS)
@pytest.mark.parametrize("prec", PRECS)
def test_every_variant_in_place(cuda, prec, direction):
    """In place (d_in == d_out) is bit-identical to out of place for every
    compiled variant -- each kernel reads its rows (registers, staging or
    tensor memory) before any store; an odd batch leaves a partial last CTA."""
    lib = sf._native.lib()
    for n in ALL_N:
        x = torch.from_numpy(sf.generate_batch(333, n, seed=12, precision=prec)).to(cuda)
        for v in range(lib.sfft_num_variants(n, 0 if prec == "single" else 1)):
            plan = sf.make_plan(n, direction, precision=prec, variant=v)
            want = torch.empty_like(x)
            sf.launch(plan, x, want, 333)
            buf = x.clone()
            sf.launch(plan, buf, buf, 333)
            torch.cuda.synchronize()
            assert torch.equal(buf, want), (n, v, direction)


def test_plan_info_and_twiddles(cuda):
    plan = sf.make_plan(2048, precision="double")
    info = plan.kernel_info(0)
    assert info["n"] == 2048 and info["precision"] == 1
    assert int(np.prod(info["radices"])) == 2048
    import ctypes

    buf = np.empty(2048, np.complex128)
    sf._native.check(sf._native.lib().sfft_plan_twiddles(plan.native_handle(0), buf.ctypes.data, buf.nbytes))
    assert np.array_equal(buf, plan.twiddles.factors)
    assert ctypes is not None


@pytest.mark.parametrize("prec,n", [("single", 2), ("single", 1024), ("double", 2048)])
def test_more_than_2_31_elements(cuda, prec, n):
    """64-bit indexing: a batch with > 2^31 complex elements (16-32 GiB each way)."""
    elems = (1 << 31) + 4096
    batch = elems // n + 3
    cdt = torch.complex64 if prec == "single" else torch.complex128
    free, _ = torch.cuda.mem_get_info()
    need = 2 * batch * n * (8 if prec == "single" else 16)
    if need > 0.8 * free:
        pytest.skip("not enough device memory")
    x = torch.empty((batch, n), dtype=cdt, device=cuda)
    x.real.uniform_(-1, 1)
    x.imag.uniform_(-1, 1)
    plan = sf.make_plan(n, precision=prec)
    y = torch.empty_like(x)
    sf.launch(plan, x, y, batch)
    rows = [0, 1, batch // 2, batch - 2, batch - 1]
    xs = x[rows].cpu().numpy()
    got = y[rows].cpu().numpy()
    del x, y
    torch.cuda.empty_cache()
    assert row_rel_l2(got, oracle.direct_dft(xs)).max() <= tolerance(n, prec)


def test_host_pipeline_shared_across_plans(cuda):
    """sfft_execute_host keeps one pipeline per device (streams, slots, pinned
    staging) shared by every plan: interleaved plans of different row sizes,
    chunked and small calls, pageable and pinned buffers, all bit-identical
    to the device path."""
    specs = [(8, "single", "forward", (40 << 20) // 64 + 7), (2048, "double", "inverse", (40 << 20) // (2048 * 16) + 3),
             (64, "single", "inverse", 100), (1024, "double", "forward", (70 << 20) // (1024 * 16) + 1),
             (2, "double", "forward", 5)]
    cases = []
    for n, prec, direction, rows in specs:
        x = sf.generate_batch(rows, n, seed=n, precision=prec)
        plan = sf.make_plan(n, direction, precision=prec)
        cases.append((plan, x, run(plan, x, cuda)))
    for rep in range(2):
        for plan, x, want in cases:
            got = sf.execute(plan, x if rep == 0 else torch.from_numpy(x).pin_memory().numpy())
            assert np.array_equal(got, want)


@pytest.mark.parametrize("prec", PRECS)
def test_nonfinite_detection_every_variant(cuda, prec):
    """The Stockham/split2 kernels test X[0] (the sum of every input) after the
    passes instead of every input; in-place launches test the inputs.  Every
    variant, both directions, NaN/Inf in the first, a middle and the last row
    of an odd batch (partial CTA), real input where supported -- and finite
    rows whose X[0] overflows must NOT raise (the reference checks inputs)."""
    lib = sf._native.lib()
    code = 0 if prec == "single" else 1
    dt = dtype_of(prec)
    big = 3.0e37 if prec == "single" else 1.0e306  # finite, but N of them overflow
    for n in ALL_N:
        for v in range(lib.sfft_num_variants(n, code)):
            info = sf._native.variant_info(n, code, v)
            for direction in DIRS:
                plan = sf.make_plan(n, direction, precision=prec, variant=v)
                for row, col, val in ((0, 0, np.inf), (150, n // 2, complex(0, np.nan)), (300, n - 1, -np.inf)):
                    x = np.ones((301, n), dt)
                    x[row, col] = val
                    xd = torch.from_numpy(x).to(cuda)
                    with pytest.raises(sf.DomainError):
                        sf.execute(plan, xd)
                    flag = torch.zeros(1, dtype=torch.int32, device=cuda)
                    buf = xd.clone()
                    sf.launch(plan, buf, buf, 301, flag=flag)  # in place
                    torch.cuda.synchronize()
                    assert int(flag.item()) == 1, (n, v, direction, row)
                    if info["real_input"] and row == 0:
                        xr = torch.ones((301, n), dtype=torch.float32 if prec == "single" else torch.float64,
                                        device=cuda)
                        xr[300, 0] = float("nan")
                        with pytest.raises(sf.DomainError):
                            sf.execute(plan, xr)
                if n >= 1024:
                    x = np.full((7, n), big, dt)
                    y = sf.execute(plan, torch.from_numpy(x).to(cuda)).cpu().numpy()
                    assert not np.isfinite(y[:, 0]).all()  # X[0] overflowed, no DomainError
