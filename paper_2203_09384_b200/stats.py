"""Spectrum agreement statistics: the reference ``stats`` module (stats.py:27-239)
plus a batched GPU form.

The paper's section 6.2 check compares two spectra through their magnitude
histograms: shared linear edges, a reduced chi-square of one histogram's
counts against the other's, the chi-square survival probability from the
regularized incomplete gamma function, and the worst elementwise relative
difference.  Per spectrum pair (``compare_spectra``) the semantics are the
reference's: same report fields in the same order, same error classes, the
same series / continued-fraction split of the incomplete gamma.

``verify_batch`` (new) runs the statistic for every row of a ``(B, N)``
result on the GPU at once -- per-row edges, counts by bucketize +
scatter-add, per-row p-values from ``torch.special.gammaincc`` -- and reports
the row with the smallest p-value.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import DomainError, InsufficientDataError, ShapeError
from .validation import as_signal, check_same_length

#: convergence tolerance and iteration cap of the incomplete-gamma expansions
GAMMA_TOL = 1e-12
GAMMA_MAX_ITER = 500

#: what the histograms are built over
BIN_SOURCES = ("magnitude", "real", "imag")

_PROJECT = {
    "magnitude": np.abs,
    "real": np.real,
    "imag": np.imag,
}


@dataclass(frozen=True, eq=False)
class Histogram:
    """Counts over bin edges shared with its partner histogram (stats.py:27-37).

    ``degenerate``: every value was equal, so the edges are one artificial
    unit-wide bin ``[v, v + 1]``.
    """

    bin_edges: np.ndarray
    counts: np.ndarray
    degenerate: bool = False


@dataclass(frozen=True)
class ChiSquareReport:
    """One spectrum comparison (stats.py:40-50; field order is part of the contract)."""

    chi2_reduced: float
    ndf: int
    p_value: float
    bins_used: int
    bins_skipped: int
    max_rel_diff: float
    abs_diff_max: float


# ------------------------------------------------------------------ histograms
def _projection(x: np.ndarray, bin_on: str) -> np.ndarray:
    try:
        project = _PROJECT[bin_on]
    except KeyError:
        raise ValueError(f"bin_on must be one of {BIN_SOURCES}, got {bin_on!r}") from None
    return np.asarray(project(x), dtype=np.float64)


def _shared_edges(lo: float, hi: float, bins: int) -> tuple[np.ndarray, bool]:
    flat = bool(lo == hi)
    edges = np.array([lo, lo + 1.0]) if flat else np.linspace(lo, hi, bins + 1)
    edges.setflags(write=False)
    return edges, flat


def build_histograms(a, b, bins: int, bin_on: str = "magnitude"):
    """``(hist_a, hist_b)`` over one set of linear edges covering both inputs (stats.py:63-90)."""
    sa, sb = as_signal(a, name="a"), as_signal(b, name="b")
    check_same_length(sa, sb, names=("a", "b"))
    if bins < 2:
        raise DomainError(f"bins must be >= 2, got {bins}")
    pa, pb = _projection(sa, bin_on), _projection(sb, bin_on)
    edges, flat = _shared_edges(min(pa.min(), pb.min()), max(pa.max(), pb.max()), int(bins))
    return tuple(Histogram(edges, np.histogram(p, bins=edges)[0].astype(np.float64), flat) for p in (pa, pb))


def chi2_reduced(sample: Histogram, reference: Histogram) -> tuple[float, int]:
    """``(chi2 / ndf, ndf)``: Pearson chi-square over bins the reference occupies (stats.py:93-110).

    chi2 = sum (s_i - n_i)^2 / n_i over n_i > 0; ndf = occupied bins - 1.
    """
    if not np.array_equal(sample.bin_edges, reference.bin_edges):
        raise ShapeError("histograms must share identical bin edges")
    occupied = np.flatnonzero(reference.counts > 0)
    if occupied.size < 2:
        raise InsufficientDataError(f"only {occupied.size} usable bin(s); need at least 2 for a chi-square")
    expected = reference.counts[occupied]
    residual = sample.counts[occupied] - expected
    ndf = int(occupied.size) - 1
    return float(np.sum(residual * residual / expected)) / ndf, ndf


# ----------------------------------------------------------- incomplete gamma
def _check_gamma_domain(a: float, x: float) -> None:
    if a <= 0:
        raise DomainError(f"gamma shape parameter must be > 0, got {a}")
    if math.isnan(x) or x < 0:
        raise DomainError(f"gamma argument must be >= 0, got {x}")


def _scale(a: float, x: float) -> float:
    """x^a e^-x / Gamma(a), the common factor of both expansions."""
    return math.exp(a * math.log(x) - x - math.lgamma(a))


def _p_by_series(a: float, x: float) -> float:
    """P(a, x) = scale * sum_k x^k / (a (a+1) ... (a+k)); converges fast for x < a + 1."""
    if x == 0.0:
        return 0.0
    term = 1.0 / a
    acc = term
    k = 0
    while k < GAMMA_MAX_ITER:
        k += 1
        term *= x / (a + k)
        acc += term
        if abs(term) < abs(acc) * GAMMA_TOL:
            return acc * _scale(a, x)
    raise ArithmeticError(f"lower incomplete gamma series did not converge for a={a}, x={x}")


def _q_by_continued_fraction(a: float, x: float) -> float:
    """Q(a, x) from the Legendre continued fraction, modified Lentz; for x >= a + 1."""
    floor = 1e-300

    def guard(v: float) -> float:
        return floor if abs(v) < floor else v

    b = x + 1.0 - a
    c = 1.0 / floor
    d = 1.0 / b
    frac = d
    for i in range(1, GAMMA_MAX_ITER + 1):
        an = -i * (i - a)
        b += 2.0
        d = 1.0 / guard(an * d + b)
        c = guard(b + an / c)
        ratio = c * d
        frac *= ratio
        if abs(ratio - 1.0) < GAMMA_TOL:
            return frac * _scale(a, x)
    raise ArithmeticError(f"upper incomplete gamma continued fraction did not converge for a={a}, x={x}")


def lower_regularized_gamma(a: float, x: float) -> float:
    """P(a, x), always by the series -- the independent counterpart of Q (stats.py:158-164)."""
    _check_gamma_domain(a, x)
    return _p_by_series(a, x)


def upper_regularized_gamma(a: float, x: float) -> float:
    """Q(a, x) = 1 - P(a, x): series below x = a + 1, continued fraction above (stats.py:167-177)."""
    _check_gamma_domain(a, x)
    if x == 0.0:
        return 1.0
    if x >= a + 1.0:
        return _q_by_continued_fraction(a, x)
    return 1.0 - _p_by_series(a, x)


def chi2_p_value(chi2_total: float, ndf: int) -> float:
    """P(chi-square with ``ndf`` freedoms >= chi2_total) = Q(ndf/2, chi2/2); 1.0 at 0 (stats.py:180-190)."""
    if ndf < 1:
        raise DomainError(f"ndf must be >= 1, got {ndf}")
    if math.isnan(chi2_total) or chi2_total < 0:
        raise DomainError(f"chi2 must be finite and >= 0, got {chi2_total}")
    return upper_regularized_gamma(0.5 * ndf, 0.5 * chi2_total)


# ---------------------------------------------------------------- comparisons
def relative_difference(a, b) -> np.ndarray:
    """|a_k - b_k| / |a_k| as float64 (stats.py:193-206).

    0 where both are zero; inf where only ``a`` is zero (flagged, not raised).
    """
    sa, sb = as_signal(a, name="a"), as_signal(b, name="b")
    check_same_length(sa, sb, names=("a", "b"))
    wa, wb = sa.astype(np.complex128), sb.astype(np.complex128)
    den = np.abs(wa)
    num = np.abs(wa - wb)
    with np.errstate(divide="ignore", invalid="ignore"):
        out = np.where(den > 0, num / np.where(den > 0, den, 1.0), np.inf)
    out[(den == 0) & (wb == 0)] = 0.0
    return out.astype(np.float64)


def compare_spectra(lhs, rhs, bins: int | None = None, bin_on: str = "magnitude") -> ChiSquareReport:
    """Agreement of spectrum ``lhs`` with reference ``rhs`` (stats.py:209-239).

    ``bins`` defaults to the spectrum length; ``rhs`` supplies the expected
    counts; relative differences are taken against ``lhs`` magnitudes.
    """
    sl, sr = as_signal(lhs, name="lhs"), as_signal(rhs, name="rhs")
    check_same_length(sl, sr, names=("lhs", "rhs"))
    nbins = sl.shape[0] if bins is None else bins
    h_lhs, h_rhs = build_histograms(sl, sr, nbins, bin_on)
    red, ndf = chi2_reduced(h_lhs, h_rhs)
    used = ndf + 1
    return ChiSquareReport(
        chi2_reduced=red,
        ndf=ndf,
        p_value=chi2_p_value(red * ndf, ndf),
        bins_used=used,
        bins_skipped=int(h_rhs.counts.size) - used,
        max_rel_diff=float(relative_difference(sl, sr).max()),
        abs_diff_max=float(np.abs(sl.astype(np.complex128) - sr.astype(np.complex128)).max()),
    )


# ------------------------------------------------------------- batched (GPU)
@dataclass(frozen=True)
class BatchReport:
    """``verify_batch`` summary: the least likely row and the batch extremes."""

    rows: int
    worst_row: int           # row with the smallest p-value
    p_value_min: float       # its p-value (a true minimum over rows)
    chi2_reduced_at_worst: float
    ndf_at_worst: int
    chi2_reduced_max: float  # largest reduced chi-square of any row
    max_rel_l2: float        # worst per-row ||out - ref|| / ||ref|| (the north-star metric)
    max_abs_diff: float


def verify_batch(out, ref, bins: int | None = None, bin_on: str = "magnitude") -> BatchReport:
    """Per-row chi-square of ``out`` against ``ref`` for a whole ``(B, N)`` batch on the GPU.

    Each row gets its own linear edges from the joint min to max of the two
    rows (as ``build_histograms``), ``bins`` (default N) bins, counts via
    bucketize + scatter-add, and a p-value Q(ndf/2, chi2/2).  Rows with
    fewer than 2 occupied reference bins have no chi-square and count as
    p = 1.
    """
    import torch

    from .oracle import _cuda_torch

    _cuda_torch()
    if bin_on not in BIN_SOURCES:
        raise ValueError(f"bin_on must be one of {BIN_SOURCES}, got {bin_on!r}")

    def as_dev(v):
        t = v if isinstance(v, torch.Tensor) else torch.from_numpy(np.asarray(v))
        return t.cuda().to(torch.complex128)

    a, b = as_dev(out), as_dev(ref)
    if a.shape != b.shape or a.ndim != 2:
        raise ShapeError(f"out and ref must be equal (B, N) arrays, got {tuple(a.shape)} and {tuple(b.shape)}")
    rows, n = a.shape
    nb = int(bins or n)
    if nb < 2:
        raise DomainError(f"bins must be >= 2, got {nb}")
    pick = {"magnitude": torch.abs, "real": torch.real, "imag": torch.imag}[bin_on]
    va, vb = pick(a).contiguous(), pick(b).contiguous()
    lo = torch.minimum(va.amin(1), vb.amin(1))[:, None]
    hi = torch.maximum(va.amax(1), vb.amax(1))[:, None]
    width = torch.where(hi > lo, (hi - lo) / nb, torch.ones_like(hi))

    def counts(v):
        idx = ((v - lo) / width).floor_().clamp_(0, nb - 1).to(torch.int64)
        return torch.zeros(rows, nb, dtype=torch.float64, device=v.device).scatter_add_(1, idx, torch.ones_like(v))

    ca, cb = counts(va), counts(vb)
    occupied = cb > 0
    ndf = occupied.sum(1) - 1
    chi2 = torch.where(occupied, (ca - cb) ** 2 / cb.clamp(min=1), torch.zeros_like(ca)).sum(1)
    has_stat = ndf >= 1
    ndf_f = ndf.clamp(min=1).to(torch.float64)
    red = torch.where(has_stat, chi2 / ndf_f, torch.zeros_like(chi2))
    p = torch.where(has_stat, torch.special.gammaincc(0.5 * ndf_f, 0.5 * chi2), torch.ones_like(chi2))
    worst = int(torch.argmin(p))
    rel = torch.linalg.vector_norm(a - b, dim=1) / torch.linalg.vector_norm(b, dim=1).clamp(min=1e-300)
    return BatchReport(
        rows=rows,
        worst_row=worst,
        p_value_min=float(p[worst]),
        chi2_reduced_at_worst=float(red[worst]),
        ndf_at_worst=int(ndf[worst].clamp(min=0)),
        chi2_reduced_max=float(red.max()),
        max_rel_l2=float(rel.max()),
        max_abs_diff=float((a - b).abs().max()),
    )
