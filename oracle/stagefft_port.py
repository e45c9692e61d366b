"""Batched numpy restatement of the reference FFT path -- TEST INFRASTRUCTURE ONLY.

Every function here re-states one piece of the reference ``stagefft``
package (``/root/reference/pkg/src/stagefft``), generalised in two ways the
GPU path needs and the reference lacks:

* a leading batch axis: arrays are ``(B, N)`` and every elementwise numpy
  expression of the reference is applied to all rows at once, which keeps
  the per-element arithmetic (and so the complex64 bits) identical to the
  reference's one-row-per-call loop (``estimator.py:61-68``);
* a precision axis: the stage kernels are dtype generic, so the same code
  runs on complex128 inputs with a complex128 table -- the fp64 oracle recipe
  of SURVEY.md section 8(c).

The product code never imports this module (see ``oracle/__init__.py``).
"""

from __future__ import annotations

import math
from enum import Enum

import numpy as np

__all__ = [
    "Direction",
    "build_twiddle_table",
    "dft_matrix",
    "digit_reversal_permutation",
    "direct_dft",
    "factorize_stages",
    "generate",
    "generate_batch",
    "mixed_radix_execute",
    "reference_execute",
    "split_radix_execute",
]

# kernels.py:25 -- the eighth-root magnitude, evaluated once in double.
_HALF_SQRT2 = float(np.sqrt(0.5))


class Direction(Enum):
    """planner.py:28-30."""

    FORWARD = "forward"
    INVERSE = "inverse"


def _pow2(n: int) -> bool:
    # numerics.py:23-25
    return n > 0 and n & (n - 1) == 0


# --------------------------------------------------------------------------
# plan-time pieces
# --------------------------------------------------------------------------

def factorize_stages(n: int, *, min_length: int = 8) -> list[int]:
    """Greedy radix-8-first factorisation (planner.py:38-59).

    ``min_length`` defaults to the reference engine floor (8); the GPU plan
    widens the range to 2, where the list degenerates to ``[n]``.
    """
    if not _pow2(n) or not min_length <= n <= 2048:
        raise ValueError(f"unsupported length {n}")
    out: list[int] = []
    rest = n
    while rest % 8 == 0:
        out.append(8)
        rest //= 8
    if rest != 1:
        out.append(rest)
    return out


def digit_reversal_permutation(stages) -> np.ndarray:
    """Mixed-radix digit reversal, last stage most significant (planner.py:62-89).

    Vectorised over all indices instead of the reference's per-index loop;
    the digit arithmetic is the same.
    """
    radices = [int(r) for r in stages]
    n = math.prod(radices)
    p = np.arange(n, dtype=np.int64)
    src = np.zeros(n, dtype=np.int64)
    weight, mult = n, 1
    for r in reversed(radices):
        weight //= r
        digit, p = np.divmod(p, weight)
        src += digit * mult
        mult *= r
    return src.astype(np.intp)


def build_twiddle_table(n: int, dtype=np.complex64) -> np.ndarray:
    """exp(-2 pi i k / n), angle in float64, rounded once (numerics.py:55-71).

    ``dtype=np.complex128`` gives the fp64 table of SURVEY.md 8(c) step 1.
    """
    k = np.arange(n, dtype=np.float64)
    theta = (-2.0 * np.pi / n) * k
    table = (np.cos(theta) + 1j * np.sin(theta)).astype(dtype)
    table[0] = 1.0 + 0.0j
    return table


# --------------------------------------------------------------------------
# the butterfly engine, batched over a leading axis
# --------------------------------------------------------------------------

def _stage_operands(data, table, radix, stride, inverse):
    """Twiddle gather + multiply of one stage (kernels.py:41-72), batched.

    ``data`` is (B, n); returns (B, n/span, radix, stride) where operand
    (q, j) of every group has been multiplied by table[(n/span)*q*j mod n].
    """
    rows, n = data.shape
    span = radix * stride
    q = np.arange(radix, dtype=np.int64)[:, None]
    j = np.arange(stride, dtype=np.int64)[None, :]
    w = table[((n // span) * q * j) % n]
    if inverse:
        w = np.conj(w)
    return data.reshape(rows, n // span, radix, stride) * w


def _four_point(a, b, c, d, rot):
    # kernels.py:98-104 (operands already twiddled; rot = -i fwd, +i inv)
    s0 = a + c
    s1 = a - c
    s2 = b + d
    s3 = rot * (b - d)
    return s0 + s2, s1 + s3, s0 - s2, s1 - s3


def _radix_stage(data, table, radix, stride, inverse):
    """One radix-2/4/8 DIT stage (kernels.py:83-151); returns (B, n) output."""
    v = _stage_operands(data, table, radix, stride, inverse)
    rot = 1j if inverse else -1j
    dst = np.empty_like(v)
    if radix == 2:
        np.add(v[:, :, 0], v[:, :, 1], out=dst[:, :, 0])
        np.subtract(v[:, :, 0], v[:, :, 1], out=dst[:, :, 1])
    elif radix == 4:
        outs = _four_point(v[:, :, 0], v[:, :, 1], v[:, :, 2], v[:, :, 3], rot)
        for slot, val in enumerate(outs):
            dst[:, :, slot] = val
    elif radix == 8:
        e = _four_point(v[:, :, 0], v[:, :, 2], v[:, :, 4], v[:, :, 6], rot)
        o0, o1, o2, o3 = _four_point(v[:, :, 1], v[:, :, 3], v[:, :, 5], v[:, :, 7], rot)
        # same constant expressions as kernels.py:139-141 so the weak-scalar
        # promotion (and therefore every bit) matches the reference
        o = (
            o0,
            (_HALF_SQRT2 * (1 + rot)) * o1,
            rot * o2,
            (_HALF_SQRT2 * (rot - 1)) * o3,
        )
        for slot in range(4):
            dst[:, :, slot] = e[slot] + o[slot]
            dst[:, :, slot + 4] = e[slot] - o[slot]
    else:
        raise ValueError(f"radix {radix}")
    return dst.reshape(data.shape)


def mixed_radix_execute(x, direction=Direction.FORWARD, stages=None, dtype=None):
    """Digit-reverse, fold the radix stages, normalise (executor.py:55-96).

    ``x`` is (B, N) or (N,); ``dtype`` picks complex64 (reference engine) or
    complex128 (fp64 oracle).  For N < 8 the stage list defaults to all
    radix-2, as in the fp64 recipe of SURVEY.md 8(c).
    """
    direction = Direction(direction)
    x = np.asarray(x)
    squeeze = x.ndim == 1
    x2 = np.atleast_2d(x)
    dtype = np.dtype(dtype or np.complex64)
    n = x2.shape[-1]
    if stages is None:
        stages = factorize_stages(n) if n >= 8 else [2] * (n.bit_length() - 1)
    table = build_twiddle_table(n, dtype)
    work = np.take(x2.astype(dtype, copy=False), digit_reversal_permutation(stages), axis=-1)
    stride = 1
    inverse = direction is Direction.INVERSE
    for radix in stages:
        work = _radix_stage(work, table, radix, stride, inverse)
        stride *= radix
    out = work.copy()
    if inverse:
        out *= 1.0 / n  # executor.py:93-94 (plan.scale = 1/N, planner.py:178)
    return out[0] if squeeze else out


def _split(x, table, n_full, inverse):
    """Batched split-radix recursion on the last axis (kernels.py:168-202)."""
    length = x.shape[-1]
    if length == 1:
        return x.copy()
    if length == 2:
        out = np.empty_like(x)
        out[..., 0] = x[..., 0] + x[..., 1]
        out[..., 1] = x[..., 0] - x[..., 1]
        return out
    quarter = length // 4
    half = _split(x[..., 0::2], table, n_full, inverse)
    odd1 = _split(x[..., 1::4], table, n_full, inverse)
    odd3 = _split(x[..., 3::4], table, n_full, inverse)
    k = np.arange(quarter, dtype=np.int64) * (n_full // length)
    w1 = table[k]
    w3 = table[(3 * k) % n_full]
    if inverse:
        w1, w3 = np.conj(w1), np.conj(w3)
    rot = 1j if inverse else -1j
    a = w1 * odd1
    b = w3 * odd3
    s = a + b
    d = rot * (a - b)
    out = np.empty_like(x)
    out[..., :quarter] = half[..., :quarter] + s
    out[..., quarter : 2 * quarter] = half[..., quarter:] + d
    out[..., 2 * quarter : 3 * quarter] = half[..., :quarter] - s
    out[..., 3 * quarter :] = half[..., quarter:] - d
    return out


def split_radix_execute(x, direction=Direction.FORWARD, dtype=None):
    """Whole-transform split radix incl. the inverse 1/n (kernels.py:205-232).

    This is the reference's only engine route for N = 2 and 4.
    """
    direction = Direction(direction)
    x = np.asarray(x)
    dtype = np.dtype(dtype or np.complex64)
    xc = x.astype(dtype, copy=False)
    n = xc.shape[-1]
    inverse = direction is Direction.INVERSE
    out = _split(xc, build_twiddle_table(n, dtype), n, inverse)
    if inverse:
        out /= n
    return out


def reference_execute(x, direction=Direction.FORWARD, dtype=None):
    """What the reference computes for a batch of rows at any supported N.

    N >= 8: the mixed-radix engine (``execute`` / ``FourierTransformer``);
    N in {2, 4}: ``split_radix_transform`` (make_plan rejects them,
    planner.py:47-51).  complex128 goes through the same stage functions
    (the fp64 recipe of SURVEY.md 8(c), which for N < 8 uses radix-2 stages).
    """
    x = np.asarray(x)
    n = x.shape[-1]
    dtype = np.dtype(dtype or np.complex64)
    if n >= 8 or dtype == np.complex128:
        return mixed_radix_execute(x, direction, dtype=dtype)
    return split_radix_execute(x, direction, dtype=dtype)


# --------------------------------------------------------------------------
# ground truth and inputs
# --------------------------------------------------------------------------

def dft_matrix(n: int, direction=Direction.FORWARD) -> np.ndarray:
    """complex128 Fourier matrix with k*m reduced mod n (oracle.py:18-30)."""
    direction = Direction(direction)
    k = np.arange(n, dtype=np.int64)
    sign = 2.0j if direction is Direction.INVERSE else -2.0j
    return np.exp((sign * np.pi / n) * (np.outer(k, k) % n))


def direct_dft(x, direction=Direction.FORWARD) -> np.ndarray:
    """O(N^2) DFT of every row in complex128, no final rounding (oracle.py:33-49)."""
    direction = Direction(direction)
    x = np.asarray(x).astype(np.complex128)
    n = x.shape[-1]
    out = x @ dft_matrix(n, direction).T
    if direction is Direction.INVERSE:
        out /= n
    return out


def generate(kind: str, n: int, seed: int = 0, dtype=np.complex64) -> np.ndarray:
    """Test signals of signalgen.py:14-41 (ramp, impulse, constant, random)."""
    kind = str(kind).lower()
    if kind == "ramp":
        return np.arange(n, dtype=np.float64).astype(dtype)
    if kind == "impulse":
        out = np.zeros(n, dtype=dtype)
        out[0] = 1.0
        return out
    if kind == "constant":
        return np.ones(n, dtype=dtype)
    if kind == "random":
        return generate_batch(1, n, seed, dtype)[0]
    raise ValueError(kind)


def generate_batch(batch: int, n: int, seed: int = 0, dtype=np.complex64) -> np.ndarray:
    """Batched Philox input; row 0 of B=1 equals generate('random', n, seed).

    Same draw order as signalgen.py:37-40 with a (2, B, N) shape.
    """
    rng = np.random.Generator(np.random.Philox(key=seed))
    parts = rng.uniform(-1.0, 1.0, size=(2, batch, n))
    return (parts[0] + 1j * parts[1]).astype(dtype)


def _philox_draws(seed: int, start: int, count: int) -> np.ndarray:
    """``count`` uniform(-1, 1) draws of ``Generator(Philox(key=seed))`` starting
    at flat draw index ``start``, without generating the ones before it.

    One Philox counter step yields 4 64-bit draws and ``advance(k)`` skips k
    steps; ``uniform`` consumes exactly one draw per double.
    """
    bg = np.random.Philox(key=seed)
    bg.advance(start // 4)
    rng = np.random.Generator(bg)
    skip = start % 4
    return rng.uniform(-1.0, 1.0, size=skip + count)[skip:]


def generate_rows(batch: int, n: int, rows, seed: int = 0, dtype=np.complex64) -> np.ndarray:
    """Rows ``rows`` of ``generate_batch(batch, n, seed, dtype)``, bit for bit,
    at a cost proportional to ``len(rows)`` -- for sampled checks of
    multi-GiB batches.  Real parts are draws [r*n, (r+1)*n) of the (2, B, N)
    stream, imaginary parts the same range offset by B*n."""
    rows = np.asarray(rows, dtype=np.int64)
    out = np.empty((rows.size, n), dtype=dtype)
    for i, r in enumerate(rows):
        re = _philox_draws(seed, int(r) * n, n)
        im = _philox_draws(seed, (batch + int(r)) * n, n)
        out[i] = (re + 1j * im).astype(dtype)
    return out

