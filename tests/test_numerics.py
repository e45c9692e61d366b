"""Twiddle tables from the native plan builder (CPU only).

sfft_build_twiddle_table is the routine sfft_plan_create uses to fill the
device tables; its complex64 output must equal the reference's
build_twiddle_table bit for bit (tests/golden/plan_constants.npz).
"""

import numpy as np
import pytest

import paper_2203_09384_b200 as sf
from paper_2203_09384_b200 import InvalidLengthError, build_twiddle_table, twiddle

ALL_N = [2**p for p in range(1, 12)]


def test_single_tables_match_reference_bits(golden):
    g = golden("plan_constants.npz")
    for p in range(13):
        assert np.array_equal(build_twiddle_table(2**p).factors, g[f"twiddle_{2**p}"])


@pytest.mark.parametrize("n", ALL_N + [4096])
def test_double_tables(n):
    t = build_twiddle_table(n, "double").factors
    k = np.arange(n)
    a = (-2.0 * np.pi / n) * k
    ref = np.cos(a) + 1j * np.sin(a)
    ref[0] = 1
    assert t.dtype == np.complex128 and t[0] == 1
    assert np.max(np.abs(t - ref)) <= 2.3e-16  # libm vs numpy: <= 1 ulp
    # the single table is the double table rounded once
    assert np.array_equal(build_twiddle_table(n).factors, t.astype(np.complex64))


def test_twiddle_values():
    assert twiddle(8, 0) == 1.0
    assert abs(twiddle(8, 4) - (-1.0)) < 1e-7
    assert abs(twiddle(8, 2) - (-1j)) < 1e-7
    r = np.sqrt(0.5)
    assert abs(twiddle(8, 1) - complex(r, -r)) < 1e-7
    assert twiddle(16, 3).dtype == np.complex64
    assert twiddle(16, 3, "double").dtype == np.complex128
    for n in (4, 8, 256):
        for k in (-3, -1, 0, 5, n, n + 7, 10 * n + 1):
            assert twiddle(n, k) == twiddle(n, k % n)
    with pytest.raises(InvalidLengthError):
        twiddle(0, 1)


@pytest.mark.parametrize("n", ALL_N)
def test_table_invariants(n):
    f = build_twiddle_table(n).factors
    np.testing.assert_allclose(np.abs(f), 1.0, atol=1e-6)
    k = np.arange(n)
    np.testing.assert_allclose(f[(-k) % n], np.conj(f), atol=1e-7)
    if n >= 4:
        q = np.arange(n // 4)
        np.testing.assert_allclose(f[q + n // 4], -1j * f[q], atol=1e-6)
        np.testing.assert_allclose(f[(3 * (q + n // 4)) % n], 1j * f[(3 * q) % n], atol=1e-6)
    for kk in np.random.default_rng(n).integers(0, n, size=16):
        assert f[kk] == twiddle(n, int(kk))


def test_table_errors_and_read_only():
    for bad in (0, -2, 3, 12, 100, 8192):
        with pytest.raises(InvalidLengthError):
            build_twiddle_table(bad)
    t = build_twiddle_table(16)
    with pytest.raises(ValueError):
        t.factors[0] = 0
    assert len(build_twiddle_table(sf.TABLE_MAX_LENGTH)) == 4096
