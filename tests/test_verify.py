"""Chi-square verification tools (paper section 6.2) and the GPU direct DFT.

CPU part mirrors the reference tests/test_stats.py (frozen quadrature
p-values, gamma identities, histogram rules); the GPU part checks naive_dft
against the CPU oracle and runs the reference acceptance criteria 2 and 3
on the GPU engine's output.
"""

import math

import numpy as np
import pytest

from paper_2203_09384_b200 import DomainError, InsufficientDataError, ShapeError
from paper_2203_09384_b200.stats import (
    Histogram,
    build_histograms,
    chi2_p_value,
    chi2_reduced,
    compare_spectra,
    lower_regularized_gamma,
    relative_difference,
    upper_regularized_gamma,
)

# (chi2_total, ndf, p) frozen from quadrature of the chi-square density
# (reference tests/test_stats.py:23-44, tools/make_fixtures.py:18-40)
QUADRATURE_P = [
    (0.5, 1, 0.4795001221869535), (1.0, 1, 0.31731050786291415), (2.0, 1, 0.1572992070502851),
    (3.0, 2, 0.2231301601484298), (0.25, 2, 0.8824969025845953), (2.0, 2, 0.36787944117144233),
    (4.5, 3, 0.21229028736013356), (1.5, 4, 0.8266414672967758), (10.0, 5, 0.07523524614651222),
    (5.0, 5, 0.4158801869955079), (7.0, 7, 0.4288798575530548), (12.0, 8, 0.15120388277664798),
    (3.0, 10, 0.9814240637778593), (15.0, 10, 0.13206185628772038), (20.0, 12, 0.0670859628790319),
    (9.5, 15, 0.8499584293767105), (30.0, 20, 0.0698536606994099), (18.0, 25, 0.8423907155804603),
    (40.0, 40, 0.4702572668392401), (55.0, 50, 0.2910103006596476),
]


@pytest.mark.parametrize("chi2_total,ndf,expected", QUADRATURE_P)
def test_p_value_matches_quadrature(chi2_total, ndf, expected):
    assert chi2_p_value(chi2_total, ndf) == pytest.approx(expected, abs=1e-8)


def test_p_value_identities():
    for ndf in (1, 2, 5, 50, 2047):
        assert chi2_p_value(0.0, ndf) == 1.0
    assert chi2_p_value(2.0, 2) == pytest.approx(math.exp(-1.0), abs=1e-10)
    rng = np.random.default_rng(2024)
    for _ in range(300):
        a, x = float(rng.uniform(0.5, 60)), float(rng.uniform(0, 100))
        assert upper_regularized_gamma(a, x) + lower_regularized_gamma(a, x) == pytest.approx(1.0, abs=1e-10)
    for bad in ((-1.0, 4), (float("nan"), 4), (1.0, 0)):
        with pytest.raises(DomainError):
            chi2_p_value(*bad)
    xs = np.linspace(0, 80, 120)
    ps = [chi2_p_value(float(x), 4) for x in xs]
    assert all(p >= q - 1e-15 for p, q in zip(ps, ps[1:]))


def test_histograms_and_chi2_rules():
    x = np.array([1j, 2j, -1j], np.complex64)
    mag, _ = build_histograms(x, x, bins=2)
    imag, _ = build_histograms(x, x, bins=2, bin_on="imag")
    assert mag.bin_edges[0] == 1.0 and imag.bin_edges[0] == -1.0
    with pytest.raises(ValueError):
        build_histograms(x, x, bins=2, bin_on="phase")
    with pytest.raises(ShapeError):
        build_histograms(np.ones(8), np.ones(4), bins=4)
    with pytest.raises(DomainError):
        build_histograms(np.ones(8), np.ones(8), bins=1)
    edges = np.array([0.0, 1.0, 2.0])
    red, ndf = chi2_reduced(Histogram(edges, np.array([4.0, 6.0])), Histogram(edges, np.array([5.0, 5.0])))
    assert ndf == 1 and red == pytest.approx(0.4)
    with pytest.raises(InsufficientDataError):
        chi2_reduced(Histogram(edges, np.array([5.0, 0.0])), Histogram(edges, np.array([5.0, 0.0])))
    with pytest.raises(ShapeError):
        chi2_reduced(Histogram(edges, np.ones(2)), Histogram(np.array([0.0, 2.0, 4.0]), np.ones(2)))


def test_relative_difference():
    out = relative_difference(np.array([2, 1, 0, 0], np.complex64), np.array([1, 1, 0, 5], np.complex64))
    assert out[0] == pytest.approx(0.5) and out[1] == 0.0 and out[2] == 0.0 and np.isinf(out[3])


def test_compare_spectra_fields_and_detection():
    from dataclasses import asdict

    import oracle

    x = oracle.generate("random", 512, 3)
    y = oracle.generate("random", 512, 4)
    rep = compare_spectra(oracle.direct_dft(x), oracle.direct_dft(y), bins=32)
    assert rep.chi2_reduced > 0.01 and rep.p_value < 0.999
    assert list(asdict(rep)) == ["chi2_reduced", "ndf", "p_value", "bins_used", "bins_skipped",
                                 "max_rel_diff", "abs_diff_max"]
    same = compare_spectra(oracle.direct_dft(x), oracle.direct_dft(x))
    assert same.chi2_reduced == 0.0 and same.p_value == 1.0


@pytest.mark.gpu
def test_naive_dft_matches_oracle(cuda):
    import oracle
    import paper_2203_09384_b200 as sf
    from paper_2203_09384_b200.oracle import naive_dft, naive_dft_batch

    for n in (1, 5, 16, 100, 2048):
        x = oracle.generate_batch(3, n, seed=n, dtype=np.complex128)
        for d in ("forward", "inverse"):
            got = naive_dft_batch(x, d, precision="double")
            want = oracle.direct_dft(x, d)
            assert np.max(np.abs(got - want)) <= 1e-9 * max(1.0, np.abs(want).max())
    assert naive_dft(np.arange(8.0)).dtype == np.complex64
    with pytest.raises(DomainError):
        naive_dft(np.array([1.0, np.nan]))
    with pytest.raises(ShapeError):  # 1-D only, as the reference (tests/test_oracle.py)
        naive_dft(np.ones((4, 4)))
    # single-precision 1-D route == the batch route's single rounding
    x = oracle.generate_batch(1, 64, seed=3, dtype=np.complex64)
    assert np.array_equal(naive_dft(x[0]), naive_dft_batch(x)[0])
    assert sf is not None


@pytest.mark.gpu
def test_acceptance_criteria_2_3_on_gpu(cuda):
    """Reference acceptance criteria 2/3 (test_acceptance.py:94-114): ramp-2048."""
    import paper_2203_09384_b200 as sf
    from paper_2203_09384_b200.oracle import naive_dft

    x = sf.generate("ramp", 2048)
    engine = sf.execute(sf.make_plan(2048), x)
    rep = compare_spectra(engine, naive_dft(x), bins=2048)
    assert rep.chi2_reduced <= 0.01 and rep.p_value >= 0.999
    assert rep.max_rel_diff <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["single", "double"])
def test_verify_batch_full_config(cuda, prec):
    """chi-square + rel-L2 over every row of a large batch, GPU vs direct DFT."""
    import torch

    import paper_2203_09384_b200 as sf
    from paper_2203_09384_b200.oracle import naive_dft_batch
    from paper_2203_09384_b200.stats import verify_batch

    n, b = 1024, 4096
    x = torch.from_numpy(sf.generate_batch(b, n, seed=9, precision=prec)).to(cuda)
    y = sf.execute(sf.make_plan(n, precision=prec), x)
    ref = naive_dft_batch(x, precision="double")
    rep = verify_batch(y, ref)
    assert rep.rows == b
    assert rep.max_rel_l2 <= (1e-5 if prec == "single" else 1e-13) * 10
    assert rep.p_value_min >= 0.999
    for bin_on in ("real", "imag"):
        assert verify_batch(y, ref, bin_on=bin_on).p_value_min >= 0.999


@pytest.mark.gpu
def test_verify_batch_reports_true_minimum_p(cuda):
    """p_value_min is the minimum over rows, not the p of the
    largest reduced chi-square (rows differ in ndf)."""
    import torch

    from paper_2203_09384_b200.stats import verify_batch

    rng = np.random.default_rng(4)
    ref = torch.from_numpy(rng.standard_normal((6, 256)) + 1j * rng.standard_normal((6, 256)))
    out = ref.clone()
    out[2] *= 1.3  # one visibly different row
    out[5, :128] *= 1.05
    rep = verify_batch(out, ref)
    ps = [verify_batch(out[i:i + 1], ref[i:i + 1]).p_value_min for i in range(6)]
    assert rep.p_value_min == pytest.approx(min(ps), rel=1e-12, abs=1e-300)
    assert rep.worst_row == int(np.argmin(ps))
    with pytest.raises(ValueError):
        verify_batch(out, ref, bin_on="phase")
