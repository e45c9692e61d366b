"""Pin the CPU oracle against the reference itself (CPU only).

tests/golden/*.npz were produced by importing the reference package
(tests/golden/make_golden.py).  The oracle port must reproduce every
reference output BIT FOR BIT -- it performs the same numpy operations batched
over rows -- and must satisfy the reference's own known-answer tests.
"""

import numpy as np
import pytest

import oracle
from conftest import rel_l2

ENGINE_N = [2**p for p in range(3, 12)]
ALL_N = [2**p for p in range(1, 12)]
KINDS = ("random", "ramp", "impulse", "constant")


@pytest.mark.parametrize("n", ENGINE_N)
def test_engine_outputs_bit_exact(golden, n):
    g = golden("engine_c64.npz")
    for kind in KINDS:
        x = g[f"in_{kind}_{n}"]
        assert np.array_equal(x, oracle.generate(kind, n, seed=n))
        for d in ("forward", "inverse"):
            ref = g[f"out_{kind}_{n}_{d}"]
            assert np.array_equal(oracle.mixed_radix_execute(x, d), ref)
            # batched: the row's bits do not depend on its neighbours
            batch = np.stack([oracle.generate("random", n, 1), x, oracle.generate("ramp", n)])
            assert np.array_equal(oracle.reference_execute(batch, d)[1], ref)


@pytest.mark.parametrize("n", [2, 4, 8, 16, 64])
def test_split_radix_bit_exact(golden, n):
    g = golden("engine_c64.npz")
    x = g[f"in_split_{n}"]
    for d in ("forward", "inverse"):
        got = oracle.split_radix_execute(np.stack([x, x]), d)
        assert np.array_equal(got[0], g[f"out_split_{n}_{d}"])
        assert np.array_equal(got[1], g[f"out_split_{n}_{d}"])


@pytest.mark.parametrize("n", ALL_N)
def test_fp64_restatement_bit_exact_and_accurate(golden, n):
    g = golden("restated_c128.npz")
    x = g[f"in_{n}"]
    for d in ("forward", "inverse"):
        got = oracle.mixed_radix_execute(x[None], d, dtype=np.complex128)[0]
        assert np.array_equal(got, g[f"out_{n}_{d}"])
        # <= 8.4e-16 vs the direct DFT; tolerance 1e-13*log2(N)
        assert rel_l2(got, oracle.direct_dft(x, d)) <= 1e-15


def test_plan_constants(golden):
    g = golden("plan_constants.npz")
    for n in ENGINE_N:
        assert oracle.factorize_stages(n) == list(g[f"stages_{n}"])
    for key in [k for k in g.files if k.startswith("perm_")]:
        stages = [int(s) for s in key[5:].split("_")]
        assert np.array_equal(oracle.digit_reversal_permutation(stages), g[key])
    for p in range(13):
        assert np.array_equal(oracle.build_twiddle_table(2**p), g[f"twiddle_{2**p}"])


def test_reference_known_answers():
    # RAMP8_SPECTRUM closed form (reference tests/test_oracle.py:9-20)
    ramp8 = np.array([28, -4 + 9.65685424949238j, -4 + 4.000000000000001j, -4 + 1.6568542494923804j,
                      -4 + 2.4492935982947064e-16j, -4 - 1.65685424949238j, -4 - 3.999999999999999j,
                      -4 - 9.656854249492376j])
    np.testing.assert_allclose(oracle.direct_dft(np.arange(8.0)), ramp8, atol=1e-12)
    np.testing.assert_allclose(oracle.mixed_radix_execute(np.arange(8.0)), ramp8, atol=1e-5)
    # PERM_8_2 (reference tests/test_planner.py:20) and bit reversal
    assert list(oracle.digit_reversal_permutation([8, 2])) == [0, 2, 4, 6, 8, 10, 12, 14, 1, 3, 5, 7, 9, 11, 13, 15]
    assert list(oracle.digit_reversal_permutation([2, 2, 2])) == [0, 4, 2, 6, 1, 5, 3, 7]
    # single butterflies and radix-4 ramp (reference tests/test_kernels.py:43-58)
    np.testing.assert_allclose(oracle.split_radix_execute(np.array([1, 1])), [2, 0], atol=1e-7)
    np.testing.assert_allclose(oracle.split_radix_execute(np.array([1, 2])), [3, -1], atol=1e-7)
    np.testing.assert_allclose(oracle.split_radix_execute(np.arange(4)), [6, -2 + 2j, -2, -2 - 2j], atol=1e-6)
    # radix-8 impulse/constant (tests/test_kernels.py:61-71)
    imp = np.zeros(8)
    imp[0] = 1
    np.testing.assert_allclose(oracle.mixed_radix_execute(imp), np.ones(8), atol=1e-6)
    np.testing.assert_allclose(oracle.mixed_radix_execute(np.ones(8)), 8 * imp, atol=1e-6)


def test_estimator_fixture(golden):
    """FourierTransformer output (per-row loop over execute) == batched oracle."""
    g = golden("estimator_c64.npz")
    assert np.array_equal(oracle.reference_execute(g["X"], "forward"), g["Y"])
    assert np.array_equal(oracle.reference_execute(g["Y"], "inverse"), g["Xback"])


def test_signal_generator(golden):
    g = golden("signals_c64.npz")
    for key in g.files:
        _, n, seed = key.split("_")
        assert np.array_equal(oracle.generate("random", int(n), int(seed)), g[key])
        # batched generator, row 0 of B=1, reproduces generate() exactly
        assert np.array_equal(oracle.generate_batch(1, int(n), int(seed))[0], g[key])


@pytest.mark.parametrize("n", ALL_N)
def test_oracle_accuracy_fp32(n):
    x = oracle.generate_batch(8, n, seed=n)
    for d in ("forward", "inverse"):
        err = rel_l2(oracle.reference_execute(x, d), oracle.direct_dft(x, d))
        assert err <= 1e-5 * np.log2(n)  # reference measured 2.9e-8 .. 1.15e-7


def test_round_trip_parseval_linearity():
    n = 512
    x = oracle.generate_batch(4, n, seed=3, dtype=np.complex128)
    fx = oracle.reference_execute(x, "forward", dtype=np.complex128)
    assert rel_l2(oracle.reference_execute(fx, "inverse", dtype=np.complex128), x) <= 1e-14
    np.testing.assert_allclose(np.sum(abs(x) ** 2, -1), np.sum(abs(fx) ** 2, -1) / n, rtol=1e-13)
    y = oracle.generate_batch(4, n, seed=4, dtype=np.complex128)
    a, b = 2.5 - 0.5j, -1.25 + 3.0j
    lhs = oracle.reference_execute(a * x + b * y, "forward", dtype=np.complex128)
    assert rel_l2(lhs, a * fx + b * oracle.reference_execute(y, "forward", dtype=np.complex128)) <= 1e-14


def test_generate_rows_matches_generate_batch():
    """oracle.generate_rows (Philox jump-ahead) reproduces sampled rows of a
    batch bit for bit -- the sampled config-shape parity tests rely on it."""
    for batch, n, seed, dt in [(7, 8, 3, np.complex64), (33, 2, 0, np.complex128), (5, 2048, 9, np.complex64),
                               (1000, 4, 2, np.complex128)]:
        full = oracle.generate_batch(batch, n, seed, dt)
        idx = [0, batch - 1, batch // 2, 1, batch // 3]
        assert np.array_equal(oracle.generate_rows(batch, n, idx, seed, dt), full[idx])
