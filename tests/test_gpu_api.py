"""Reference-facing API on the GPU: estimator, execute_timed, acceptance criteria, sharding."""

import numpy as np
import pytest

import oracle
import paper_2203_09384_b200 as sf
from conftest import rel_l2, row_rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ENGINE_N = [2**p for p in range(3, 12)]


def signals(rows, width, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, (rows, width)) + 1j * rng.uniform(-1, 1, (rows, width))).astype(np.complex64)


def test_fit_transform_is_one_launch_and_bit_equal_to_execute(cuda):
    X = signals(5, 64)
    out = sf.FourierTransformer().fit_transform(X)
    plan = sf.make_plan(64)
    for row_in, row_out in zip(X, out):
        assert np.array_equal(row_out, sf.execute(plan, row_in))  # test_estimator.py:16-23


def test_estimator_golden_fixture(cuda, golden):
    g = golden("estimator_c64.npz")
    est = sf.FourierTransformer().fit(g["X"])
    Y = est.transform(g["X"])
    assert rel_l2(Y, g["Y"]) <= 1e-5 * 6
    assert rel_l2(est.inverse_transform(Y), g["Xback"]) <= 1e-5 * 6


def test_estimator_round_trips_and_params(cuda):
    X = signals(3, 128)
    est = sf.FourierTransformer().fit(X)
    assert rel_l2(est.inverse_transform(est.transform(X)), X) <= 1e-4
    X = signals(2, 32, seed=5)
    mixed = sf.FourierTransformer(algorithm="mixed").fit_transform(X)
    split = sf.FourierTransformer(algorithm="split").fit_transform(X)
    assert rel_l2(mixed, split) <= 1e-4
    X = signals(2, 16, seed=6)
    back = sf.FourierTransformer().fit(X).transform(sf.FourierTransformer(direction="inverse").fit(X).transform(X))
    assert rel_l2(back, X) <= 1e-4
    est = sf.FourierTransformer().fit(signals(2, 64))
    with pytest.raises(sf.ShapeError):
        est.transform(signals(2, 32))
    from sklearn.pipeline import Pipeline

    assert Pipeline([("fft", sf.FourierTransformer())]).fit_transform(signals(4, 8)).shape == (4, 8)
    Xd = sf.generate_batch(7, 2048, seed=1, precision="double")
    yd = sf.FourierTransformer(precision="double").fit_transform(torch.from_numpy(Xd).to(cuda))
    assert row_rel_l2(yd.cpu().numpy(), oracle.direct_dft(Xd)).max() <= 1e-13 * 11


def test_execute_timed(cuda):
    plan = sf.make_plan(512)
    x = sf.generate("ramp", 512)
    timed = sf.execute_timed(plan, x)
    # the timed output is checked against the oracle, not against execute()
    assert rel_l2(timed.output, oracle.reference_execute(x[None], "forward")[0]) <= 9e-5
    assert timed.dispatch_us >= 0.0 and timed.compute_us > 0.0
    xb = sf.generate_batch(1000, 512, seed=2)
    xt = torch.from_numpy(xb).to(cuda)
    t2 = sf.execute_timed(plan, xt)
    assert row_rel_l2(t2.output.cpu().numpy(), oracle.reference_execute(xb, "forward")).max() <= 9e-5
    assert t2.compute_us > 0
    # host input: compute covers the whole native pipeline (H2D + kernel + D2H)
    t4 = sf.execute_timed(plan, xb)
    assert isinstance(t4.output, np.ndarray) and np.array_equal(t4.output, t2.output.cpu().numpy())
    assert t4.compute_us > 0 and t4.dispatch_us >= 0
    t3 = sf.execute_timed(sf.make_plan(2048), sf.generate("ramp", 2048))
    assert t3.compute_us < 50_000  # reference soft guard (test_executor.py:121-127)


def test_criterion_01_oracle_sweep(cuda):
    worst = 0.0
    for n in ENGINE_N:
        plan = sf.make_plan(n)
        for kind in ("ramp", "impulse", "constant", "random"):
            x = sf.generate(kind, n, seed=0)
            worst = max(worst, rel_l2(sf.execute(plan, x), oracle.direct_dft(x)))
    assert worst <= 1e-4


def test_criterion_04_round_trips_batched(cuda):
    # 100 seeds per length and algorithm, as ONE batched launch per plan
    for n in ENGINE_N:
        x = np.stack([sf.generate("random", n, seed=s) for s in range(100)])
        for alg in ("mixed", "split"):
            fwd = sf.make_plan(n, "forward", alg)
            inv = sf.make_plan(n, "inverse", alg)
            assert row_rel_l2(sf.execute(inv, sf.execute(fwd, x)), x).max() <= 1e-4


def test_criterion_05_parseval_linearity(cuda):
    for n in (8, 64, 512, 2048):
        plan = sf.make_plan(n)
        rng = np.random.default_rng(n)
        a = (rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)).astype(np.complex64)
        b = (rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)).astype(np.complex64)
        fa = sf.execute(plan, a).astype(np.complex128)
        fb = sf.execute(plan, b).astype(np.complex128)
        et = float(np.sum(np.abs(a.astype(np.complex128)) ** 2))
        assert abs(et - float(np.sum(np.abs(fa) ** 2)) / n) / et <= 1e-4
        al, be = 2.5 - 0.5j, -1.25 + 3.0j
        mixed = sf.execute(plan, al * a + be * b).astype(np.complex128)
        assert rel_l2(mixed, al * fa + be * fb) <= 1e-4


def test_criterion_10_cross_plan_equivalence(cuda):
    plans = [sf.make_plan(16, stages=[8, 2]), sf.make_plan(16, stages=[4, 4]),
             sf.make_plan(16, stages=[2, 2, 2, 2]), sf.make_plan(16, algorithm="split")]
    x = np.stack([sf.generate("random", 16, seed=s) for s in range(100)])
    outs = [sf.execute(p, x) for p in plans]
    for o in outs[1:]:
        assert row_rel_l2(o, outs[0]).max() <= 1e-4


def test_split_radix_transform_on_gpu(cuda, golden):
    g = golden("engine_c64.npz")
    for n in (2, 4, 8, 16, 64):
        x = g[f"in_split_{n}"]
        for d in ("forward", "inverse"):
            y = sf.split_radix_transform(x, sf.build_twiddle_table(n), d, verify_twiddles=True)
            assert rel_l2(y, g[f"out_split_{n}_{d}"]) <= 1e-5 * max(1, np.log2(n))


def test_execute_sharded_matches_single_device(cuda):
    x = sf.generate_batch(1001, 256, seed=4)
    plan = sf.make_plan(256)
    want = sf.execute(plan, x)
    ndev = torch.cuda.device_count()
    devices = list(range(ndev)) if ndev > 1 else [0, 0, 0]
    assert np.array_equal(sf.execute_sharded(plan, x, devices), want)


def test_large_full_size_properties(cuda):
    """Config 2 at full size: round trip + Parseval over all 65536 rows on the GPU."""
    n, b = 1024, 65536
    x = torch.from_numpy(sf.generate_batch(b, n, seed=1)).to(cuda)
    y = sf.execute(sf.make_plan(n), x)
    back = sf.execute(sf.make_plan(n, "inverse"), y)
    err = (torch.linalg.vector_norm(back - x, dim=1) / torch.linalg.vector_norm(x, dim=1)).max().item()
    assert err <= 1e-5 * 10
    ex = torch.sum(torch.abs(x.to(torch.complex128)) ** 2, dim=1)
    ey = torch.sum(torch.abs(y.to(torch.complex128)) ** 2, dim=1) / n
    assert ((ex - ey).abs() / ex).max().item() <= 1e-5


@pytest.mark.parametrize("n,prec", [(1024, "single"), (2048, "double"), (8, "single")])
def test_launch_is_cuda_graph_capturable(cuda, n, prec):
    """`launch` only enqueues work on the given stream, so a chain of
    transforms (forward then inverse here) can be captured once into a CUDA
    graph and replayed -- the launch-bound way to run many small batches."""
    x = torch.from_numpy(sf.generate_batch(33, n, seed=3, precision=prec)).to(cuda)
    y, z = torch.empty_like(x), torch.empty_like(x)
    fwd = sf.make_plan(n, "forward", precision=prec)
    inv = sf.make_plan(n, "inverse", precision=prec)
    s = torch.cuda.Stream(cuda)
    with torch.cuda.stream(s):  # native plans + kernel attributes exist before capture
        sf.launch(fwd, x, y, 33, stream=s)
        sf.launch(inv, y, z, 33, stream=s)
    s.synchronize()
    want_y, want_z = y.clone(), z.clone()
    y.zero_()
    z.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sf.launch(fwd, x, y, 33, stream=s)
        sf.launch(inv, y, z, 33, stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want_y) and torch.equal(z, want_z)
    tol = (1e-5 if prec == "single" else 1e-13) * np.log2(n)
    assert rel_l2(z.cpu().numpy(), x.cpu().numpy()) <= 2 * tol


@pytest.mark.parametrize("n,prec", [(1024, "single"), (2048, "double"), (16, "single"), (8, "double")])
def test_back_to_back_launch_chain_stays_ordered(cuda, n, prec):
    """Launches on one stream use programmatic dependent launch: kernel k+1 is
    scheduled while kernel k drains and waits (griddepcontrol.wait) before
    touching memory.  A long in-place forward/inverse chain on one buffer --
    every kernel reading what the previous one wrote -- must round-trip."""
    rows = (64 << 20) // (n * (8 if prec == "single" else 16))
    x0 = torch.from_numpy(sf.generate_batch(rows, n, seed=9, precision=prec)).to(cuda)
    buf = x0.clone()
    fwd = sf.make_plan(n, "forward", precision=prec)
    inv = sf.make_plan(n, "inverse", precision=prec)
    for _ in range(10):
        sf.launch(fwd, buf, buf, rows)
        sf.launch(inv, buf, buf, rows)
    torch.cuda.synchronize()
    tol = (1e-5 if prec == "single" else 1e-13) * np.log2(n)
    assert row_rel_l2(buf.cpu().numpy(), x0.cpu().numpy()).max() <= 20 * tol


@pytest.mark.parametrize("prec", ["single", "double"])
@pytest.mark.parametrize("n", [8, 32, 64, 1024, 2048])
def test_real_input_path(cuda, n, prec):
    """Real rows go to the kernel as reals where its loader supports it
    (sfft_execute_ex, SFFT_INPUT_REAL) -- bit-identical to widening to
    complex first, as the reference does (executor.py:74,
    tests/test_executor.py:89-92)."""
    rdt = torch.float32 if prec == "single" else torch.float64
    cdt = torch.complex64 if prec == "single" else torch.complex128
    g = torch.Generator(device=cuda).manual_seed(n)
    xr = torch.rand((777, n), generator=g, device=cuda, dtype=rdt) * 2 - 1
    for direction in ("forward", "inverse"):
        plan = sf.make_plan(n, direction, precision=prec)
        got = sf.execute(plan, xr)
        want = sf.execute(plan, xr.to(cdt))
        assert got.dtype == cdt and torch.equal(got, want)
        assert torch.equal(sf.execute(plan, xr[5]), want[5])  # 1-D
        if plan.supports_real_input(cuda.index):
            y = torch.empty((777, n), dtype=cdt, device=cuda)
            sf.launch(plan, xr, y, 777)
            torch.cuda.synchronize()
            assert torch.equal(y, want)
    # other real dtypes are cast to the plan's real type first
    plan = sf.make_plan(n, precision=prec)
    xi = torch.randint(-5, 5, (33, n), device=cuda, dtype=torch.int32)
    assert torch.equal(sf.execute(plan, xi), sf.execute(plan, xi.to(cdt)))
    bad = xr.clone()
    bad[-1, -1] = float("inf")
    with pytest.raises(sf.DomainError):
        sf.execute(plan, bad)


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_real_numpy_input_host_path(cuda, prec, pinned):
    """Real numpy rows cross the host link as reals (sfft_execute_host_ex,
    SFFT_INPUT_REAL: half the H2D bytes) -- small-call and chunked pipeline
    paths -- bit-identical to widening on the host first."""
    n = 1024
    rdt = np.float32 if prec == "single" else np.float64
    plan = sf.make_plan(n, precision=prec)
    for rows in (3, (48 << 20) // (n * 2 * np.dtype(rdt).itemsize) + 7):  # small call, > 1 chunk
        x = np.random.default_rng(rows).uniform(-1, 1, (rows, n)).astype(rdt)
        if pinned:
            x = torch.from_numpy(x).pin_memory().numpy()
        got = sf.execute(plan, x)
        want = sf.execute(plan, x.astype(plan.dtype))
        assert got.dtype == plan.dtype and got.shape == x.shape
        assert np.array_equal(got, want)
    assert np.array_equal(sf.execute_sharded(plan, x, [0, 0]), want)


@pytest.mark.parametrize("prec", ["single", "double"])
def test_real_input_every_real_capable_variant(cuda, prec):
    """Every compiled variant with a real-input loader (LDG or bulk TMA, any
    R) is bit-identical to widening, on odd batches (partial CTAs)."""
    lib = sf._native.lib()
    code = 0 if prec == "single" else 1
    rdt = torch.float32 if prec == "single" else torch.float64
    cdt = torch.complex64 if prec == "single" else torch.complex128
    checked = 0
    for p in range(1, 12):
        n = 2**p
        for v in range(lib.sfft_num_variants(n, code)):
            if not sf._native.variant_info(n, code, v)["real_input"]:
                continue
            xr = torch.rand((301, n), device=cuda, dtype=rdt) * 2 - 1
            for direction in ("forward", "inverse"):
                plan = sf.make_plan(n, direction, precision=prec, variant=v)
                y = torch.empty((301, n), dtype=cdt, device=cuda)
                sf.launch(plan, xr, y, 301)
                torch.cuda.synchronize()
                assert torch.equal(y, sf.execute(plan, xr.to(cdt))), (n, v, direction)
                checked += 1
    assert checked >= 2 * 11


@pytest.mark.parametrize("prec", ["single", "double"])
def test_zero_copy_small_calls(cuda, prec):
    """Host calls of <= 1 MiB output run the kernel on page-locked, host-mapped
    memory (sfft_execute_host zero-copy path): pageable or pinned input and
    output in every combination, in place on a pinned buffer, and real rows
    -- bit-identical to the device path, at every N, from one row up to the
    1 MiB limit and one row past it (the copy-engine path)."""
    import itertools

    esize = 8 if prec == "single" else 16
    for p in range(1, 12):
        n = 2**p
        plan = sf.make_plan(n, precision=prec)
        for rows in (1, 5, (1 << 20) // (n * esize), (1 << 20) // (n * esize) + 1):
            x = sf.generate_batch(rows, n, seed=p + rows, precision=prec)
            want = sf.execute(plan, torch.from_numpy(x).to(cuda)).cpu().numpy()
            for pin_in, pin_out in itertools.product((False, True), repeat=2):
                xi = torch.from_numpy(x.copy()).pin_memory().numpy() if pin_in else x.copy()
                out = (torch.empty(x.shape, dtype=torch.from_numpy(x).dtype, pin_memory=True).numpy()
                       if pin_out else np.empty_like(x))
                got = sf.execute(plan, xi, out=out)
                assert got is out and np.array_equal(got, want), (n, rows, pin_in, pin_out)
                assert np.array_equal(xi, x)  # the input is never written
            buf = torch.from_numpy(x.copy()).pin_memory().numpy()
            sf.execute(plan, buf, out=buf)  # in place, both sides mapped
            assert np.array_equal(buf, want), (n, rows)
        xr = np.ascontiguousarray(x.real)
        xr_pinned = torch.from_numpy(xr).pin_memory().numpy()
        want_r = sf.execute(plan, xr.astype(plan.dtype))
        assert np.array_equal(sf.execute(plan, xr_pinned), want_r)
        bad = x.copy()
        bad[-1, -1] = np.nan
        with pytest.raises(sf.DomainError):
            sf.execute(plan, torch.from_numpy(bad).pin_memory().numpy())


@pytest.mark.parametrize("prec", ["single", "double"])
def test_device_resident_shards(cuda, prec):
    """scatter_rows -> execute_shards -> gather_rows (shards stay
    resident per device, one launch each, optional gather to one device):
    bit-identical to one execute of the whole batch, for uneven splits and
    more devices than rows; NaN/Inf in any shard raises DomainError."""
    n = 512
    plan = sf.make_plan(n, precision=prec)
    for rows, devices in ((1001, [0, 0, 0]), (2, [0, 0, 0, 0]), (4096, [0])):
        x = torch.from_numpy(sf.generate_batch(rows, n, seed=rows, precision=prec)).to(cuda)
        want = sf.execute(plan, x)
        shards = sf.scatter_rows(x, devices)
        assert len(shards) == min(rows, len(devices))
        outs = sf.execute_shards(plan, shards)
        assert all(o.device == s.device for o, s in zip(outs, shards))
        assert torch.equal(sf.gather_rows(outs, 0), want)
        host = sf.scatter_rows(x.cpu().numpy(), devices)  # from host rows too
        assert torch.equal(sf.gather_rows(sf.execute_shards(plan, host), 0), want)
    bad = x.clone()
    bad[-1, 3] = float("nan")
    with pytest.raises(sf.DomainError):
        sf.execute_shards(plan, sf.scatter_rows(bad, [0, 0]))
