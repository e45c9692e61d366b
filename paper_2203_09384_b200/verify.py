"""Verification after the path: direct-DFT ground truth and chi-square agreement.

Mirror of the reference ``oracle`` (oracle.py:18-49) and ``stats``
(stats.py:27-239) modules, the paper's section 6.2 method, re-designed for
batches:

* ``dft_matrix`` / ``naive_dft`` build the O(N^2) ground truth as a complex128
  matrix product on the GPU (one ZGEMM for a whole batch), with the phase
  index k*m reduced mod N and one final rounding, exactly as oracle.py does
  row by row on the CPU.  This is the checker, not the FFT path.
* ``compare_spectra`` is the reference report for one spectrum pair
  (magnitude histograms on shared linear edges, reduced chi-square against
  the reference counts, p-value from the regularized incomplete gamma
  function, worst elementwise relative difference).
* ``verify_batch`` runs the same statistic for every row of a (B, N) result
  at once on the GPU (histograms via bucketize + scatter-add) and reports the
  worst row.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import DomainError, InsufficientDataError, InvalidLengthError, ShapeError
from .planner import Direction

GAMMA_TOL = 1e-12
GAMMA_MAX_ITER = 500
BIN_SOURCES = ("magnitude", "real", "imag")


def _torch():
    import torch

    if not torch.cuda.is_available():
        from .errors import CudaError

        raise CudaError("verify.naive_dft runs on the GPU; no CUDA device is visible")
    return torch


# ------------------------------------------------------------------ oracle
def dft_matrix(n: int, direction=Direction.FORWARD, device=None):
    """n x n complex128 Fourier matrix, exp(-+2 pi i (k m mod n) / n) (oracle.py:18-30)."""
    if n < 1:
        raise InvalidLengthError(f"transform length must be >= 1, got {n}")
    torch = _torch()
    direction = Direction(direction)
    k = torch.arange(n, dtype=torch.int64, device=device or "cuda")
    phase = torch.outer(k, k) % n
    sign = 1.0 if direction is Direction.INVERSE else -1.0
    angle = phase.to(torch.float64) * (sign * 2.0 * math.pi / n)
    return torch.polar(torch.ones_like(angle), angle)


def naive_dft(signal, direction=Direction.FORWARD, *, precision: str = "single"):
    """Direct DFT of a row or a (B, N) batch, accumulated in complex128.

    forward X[k] = sum_m x[m] w^(k m); inverse divides by n (oracle.py:33-49).
    The result is rounded once to the requested precision ("single" like the
    reference, or "double" / None for the unrounded complex128).
    """
    torch = _torch()
    direction = Direction(direction)
    is_tensor = isinstance(signal, torch.Tensor)
    x = signal if is_tensor else torch.from_numpy(np.asarray(signal))
    if x.ndim not in (1, 2) or x.shape[-1] == 0:
        raise ShapeError(f"signal must be (N,) or (B, N) and non-empty, got {tuple(x.shape)}")
    if not (x.is_complex() or x.is_floating_point() or x.dtype in (torch.int32, torch.int64)):
        raise DomainError(f"signal has non-numeric dtype {x.dtype}")
    dev = x.device if x.is_cuda else torch.device("cuda")
    xc = x.to(dev).to(torch.complex128)
    if not bool(torch.isfinite(torch.view_as_real(xc)).all()):
        raise DomainError("signal contains NaN or Inf values")
    n = xc.shape[-1]
    out = xc @ dft_matrix(n, direction, dev).T
    if direction is Direction.INVERSE:
        out = out / n
    if precision == "single":
        out = out.to(torch.complex64)
    if is_tensor:
        return out if x.is_cuda else out.cpu()
    return out.cpu().numpy()


# ------------------------------------------------------------ chi-square tools
@dataclass(frozen=True, eq=False)
class Histogram:
    """Counts over shared edges; ``degenerate`` = all values equal (stats.py:27-37)."""

    bin_edges: np.ndarray
    counts: np.ndarray
    degenerate: bool = False


@dataclass(frozen=True)
class ChiSquareReport:
    """stats.py:40-50, same field order."""

    chi2_reduced: float
    ndf: int
    p_value: float
    bins_used: int
    bins_skipped: int
    max_rel_diff: float
    abs_diff_max: float


def _as_row(values, name):
    arr = np.asarray(values)
    if arr.ndim != 1:
        raise ShapeError(f"{name} must be one-dimensional, got shape {arr.shape}")
    if arr.size == 0:
        raise InvalidLengthError(f"{name} is empty")
    if arr.dtype.kind not in "fciu":
        raise DomainError(f"{name} has non-numeric dtype {arr.dtype}")
    if not np.all(np.isfinite(arr)):
        raise DomainError(f"{name} contains NaN or Inf values")
    # single precision unless the caller hands double-precision data (the
    # reference always works in complex64, validation.py:26)
    wide = arr.dtype in (np.complex128, np.float64)
    return arr.astype(np.complex128 if wide else np.complex64)


def _values(x, bin_on):
    if bin_on == "magnitude":
        return np.abs(x).astype(np.float64)
    if bin_on == "real":
        return x.real.astype(np.float64)
    if bin_on == "imag":
        return x.imag.astype(np.float64)
    raise ValueError(f"bin_on must be one of {BIN_SOURCES}, got {bin_on!r}")


def build_histograms(a, b, bins: int, bin_on: str = "magnitude"):
    """Two histograms over one set of linear edges spanning both inputs (stats.py:63-90)."""
    xa, xb = _as_row(a, "a"), _as_row(b, "b")
    if xa.shape != xb.shape:
        raise ShapeError(f"a and b lengths differ: {xa.shape[0]} vs {xb.shape[0]}")
    if bins < 2:
        raise DomainError(f"bins must be >= 2, got {bins}")
    va, vb = _values(xa, bin_on), _values(xb, bin_on)
    lo, hi = min(va.min(), vb.min()), max(va.max(), vb.max())
    degenerate = bool(lo == hi)
    edges = np.array([lo, lo + 1.0]) if degenerate else np.linspace(lo, hi, bins + 1)
    edges.setflags(write=False)
    return tuple(
        Histogram(edges, np.histogram(v, bins=edges)[0].astype(np.float64), degenerate) for v in (va, vb)
    )


def chi2_reduced(sample: Histogram, reference: Histogram):
    """(chi2/ndf, ndf) over bins where the reference count is > 0 (stats.py:93-110)."""
    if not np.array_equal(sample.bin_edges, reference.bin_edges):
        raise ShapeError("histograms must share identical bin edges")
    used = reference.counts > 0
    n_used = int(used.sum())
    if n_used < 2:
        raise InsufficientDataError(f"only {n_used} usable bin(s); need at least 2 for a chi-square")
    d = sample.counts[used] - reference.counts[used]
    return float(np.sum(d * d / reference.counts[used])) / (n_used - 1), n_used - 1


def _gamma_prefactor(a, x):
    return math.exp(a * math.log(x) - x - math.lgamma(a))


def _p_series(a, x):
    """Regularized lower gamma P(a, x) by its power series."""
    if x == 0.0:
        return 0.0
    term = total = 1.0 / a
    ap = a
    for _ in range(GAMMA_MAX_ITER):
        ap += 1.0
        term *= x / ap
        total += term
        if abs(term) < abs(total) * GAMMA_TOL:
            return total * _gamma_prefactor(a, x)
    raise ArithmeticError(f"gamma series did not converge (a={a}, x={x})")


def _q_fraction(a, x):
    """Regularized upper gamma Q(a, x) by the modified-Lentz continued fraction."""
    eps = 1e-300
    b = x + 1.0 - a
    c = 1.0 / eps
    d = 1.0 / b
    h = d
    for i in range(1, GAMMA_MAX_ITER + 1):
        an = -i * (i - a)
        b += 2.0
        d = an * d + b
        d = eps if abs(d) < eps else d
        c = b + an / c
        c = eps if abs(c) < eps else c
        d = 1.0 / d
        step = d * c
        h *= step
        if abs(step - 1.0) < GAMMA_TOL:
            return h * _gamma_prefactor(a, x)
    raise ArithmeticError(f"gamma continued fraction did not converge (a={a}, x={x})")


def _check_gamma_args(a, x):
    if a <= 0:
        raise DomainError(f"gamma shape parameter must be > 0, got {a}")
    if x < 0 or math.isnan(x):
        raise DomainError(f"gamma argument must be >= 0, got {x}")


def lower_regularized_gamma(a: float, x: float) -> float:
    """P(a, x), always by the series (stats.py:158-164)."""
    _check_gamma_args(a, x)
    return _p_series(a, x)


def upper_regularized_gamma(a: float, x: float) -> float:
    """Q(a, x): series below x = a + 1, continued fraction above (stats.py:167-177)."""
    _check_gamma_args(a, x)
    if x == 0.0:
        return 1.0
    return 1.0 - _p_series(a, x) if x < a + 1.0 else _q_fraction(a, x)


def chi2_p_value(chi2_total: float, ndf: int) -> float:
    """Survival function Q(ndf/2, chi2/2); exactly 1.0 at chi2 = 0 (stats.py:180-190)."""
    if ndf < 1:
        raise DomainError(f"ndf must be >= 1, got {ndf}")
    if math.isnan(chi2_total) or chi2_total < 0:
        raise DomainError(f"chi2 must be finite and >= 0, got {chi2_total}")
    return upper_regularized_gamma(ndf / 2.0, chi2_total / 2.0)


def relative_difference(a, b) -> np.ndarray:
    """|a_k - b_k| / |a_k|; 0 where both are 0, inf where only a is (stats.py:193-206)."""
    xa, xb = _as_row(a, "a"), _as_row(b, "b")
    if xa.shape != xb.shape:
        raise ShapeError(f"a and b lengths differ: {xa.shape[0]} vs {xb.shape[0]}")
    xa, xb = xa.astype(np.complex128), xb.astype(np.complex128)
    num, den = np.abs(xa - xb), np.abs(xa)
    out = np.full(den.shape, np.inf)
    np.divide(num, den, out=out, where=den > 0)
    out[(den == 0) & (np.abs(xb) == 0)] = 0.0
    return out


def compare_spectra(lhs, rhs, bins: int | None = None, bin_on: str = "magnitude") -> ChiSquareReport:
    """Agreement report of ``lhs`` against reference ``rhs`` (stats.py:209-239)."""
    xa, xb = _as_row(lhs, "lhs"), _as_row(rhs, "rhs")
    if xa.shape != xb.shape:
        raise ShapeError(f"lhs and rhs lengths differ: {xa.shape[0]} vs {xb.shape[0]}")
    ha, hb = build_histograms(xa, xb, bins or xa.shape[0], bin_on)
    reduced, ndf = chi2_reduced(ha, hb)
    return ChiSquareReport(
        chi2_reduced=reduced,
        ndf=ndf,
        p_value=chi2_p_value(reduced * ndf, ndf),
        bins_used=ndf + 1,
        bins_skipped=int(hb.counts.shape[0]) - (ndf + 1),
        max_rel_diff=float(relative_difference(xa, xb).max()),
        abs_diff_max=float(np.abs(xa.astype(np.complex128) - xb.astype(np.complex128)).max()),
    )


@dataclass(frozen=True)
class BatchReport:
    """Worst-row summary of ``verify_batch``."""

    rows: int
    worst_row: int
    chi2_reduced_max: float
    ndf_at_worst: int
    p_value_min: float
    max_rel_l2: float
    max_abs_diff: float


def verify_batch(out, ref, bins: int | None = None) -> BatchReport:
    """Per-row chi-square of |out| against |ref| for a whole (B, N) batch, on the GPU.

    Edges are linear per row from the row's joint min to max (as
    build_histograms); counts come from bucketize + scatter_add, so a
    65536-row batch is one pass.  Also reports the worst per-row rel-L2 and
    absolute difference (the north star's tolerance metric).
    """
    torch = _torch()
    a = out if isinstance(out, torch.Tensor) else torch.from_numpy(np.asarray(out))
    b = ref if isinstance(ref, torch.Tensor) else torch.from_numpy(np.asarray(ref))
    a, b = a.cuda().to(torch.complex128), b.cuda().to(torch.complex128)
    if a.shape != b.shape or a.ndim != 2:
        raise ShapeError(f"out and ref must be equal (B, N) arrays, got {tuple(a.shape)} and {tuple(b.shape)}")
    rows, n = a.shape
    nb = bins or n
    va, vb = a.abs(), b.abs()
    lo = torch.minimum(va.min(1).values, vb.min(1).values)[:, None]
    hi = torch.maximum(va.max(1).values, vb.max(1).values)[:, None]
    width = torch.where(hi > lo, (hi - lo) / nb, torch.ones_like(hi))

    def counts(v):
        idx = torch.clamp(((v - lo) / width).floor().to(torch.int64), 0, nb - 1)
        c = torch.zeros(rows, nb, dtype=torch.float64, device=v.device)
        return c.scatter_add_(1, idx, torch.ones_like(v))

    ca, cb = counts(va), counts(vb)
    used = cb > 0
    ndf = used.sum(1) - 1
    chi2 = torch.where(used, (ca - cb) ** 2 / cb.clamp(min=1), torch.zeros_like(ca)).sum(1)
    red = chi2 / ndf.clamp(min=1)
    rel = torch.linalg.vector_norm(a - b, dim=1) / torch.linalg.vector_norm(b, dim=1).clamp(min=1e-300)
    worst = int(torch.argmax(red))
    ndf_w = int(ndf[worst])
    red_w = float(red[worst])
    return BatchReport(
        rows=rows,
        worst_row=worst,
        chi2_reduced_max=red_w,
        ndf_at_worst=ndf_w,
        p_value_min=chi2_p_value(red_w * ndf_w, ndf_w) if ndf_w >= 1 else 1.0,
        max_rel_l2=float(rel.max()),
        max_abs_diff=float((a - b).abs().max()),
    )
