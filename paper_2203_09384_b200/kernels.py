"""Algorithm-level entry points of the reference ``kernels`` module.

Mirror of kernels.py:205-258.  The reference's butterfly engine (per-stage
radix-2/4/8 numpy passes and the split-radix recursion) is replaced by the
fused sm_100a kernels: both algorithms compute the same DFT, so
``split_radix_transform`` runs the plan's GPU kernel (one launch, no
recursion) and ``count_butterflies`` keeps the reference's arithmetic
bookkeeping.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

from .errors import InvalidLengthError, PlanError
from .numerics import TwiddleTable, is_power_of_two
from .planner import Algorithm, Direction, FftPlan, make_plan


@lru_cache(maxsize=None)
def _split_pairs(n: int) -> int:
    # B(1) = 0, B(2) = 1, B(n) = B(n/2) + 2*B(n/4) + 3n/4  (kernels.py:235-245)
    if n <= 1:
        return 0
    if n == 2:
        return 1
    return _split_pairs(n // 2) + 2 * _split_pairs(n // 4) + 3 * (n // 4)


def count_butterflies(plan: FftPlan) -> int:
    """Two-input add/subtract pairs of the plan's algorithm (kernels.py:248-258).

    Both algorithms land on (n/2)*log2(n); the GPU executes the same DFT with
    radix-8/16 passes whose in-register networks perform exactly these pairs.
    """
    if plan.algorithm is Algorithm.SPLIT_RADIX:
        return _split_pairs(plan.length)
    return sum((plan.length // 2) * (int(r).bit_length() - 1) for r in plan.stages)


def _check_quarter_turns(factors: np.ndarray) -> None:
    """w[k + n/4] = -i w[k] and w[3(k + n/4)] = +i w[3k] (kernels.py:154-165)."""
    n = factors.shape[0]
    if n < 4:
        return
    f = factors.astype(np.complex128)
    k = np.arange(n // 4)
    if not np.allclose(f[k + n // 4], -1j * f[k], atol=1e-6):
        raise AssertionError("quarter-turn identity failed (w^k)")
    if not np.allclose(f[(3 * (k + n // 4)) % n], 1j * f[(3 * k) % n], atol=1e-6):
        raise AssertionError("quarter-turn identity failed (w^3k)")


def split_radix_transform(
    signal,
    twiddles: TwiddleTable,
    direction: Direction = Direction.FORWARD,
    *,
    verify_twiddles: bool = False,
):
    """Whole transform of one signal or a batch (kernels.py:205-232).

    Accepts what the reference accepts (1-D numeric input, length a power of
    two, a table of the same length) plus ``(B, N)`` batches and CUDA
    tensors; the inverse includes the 1/N normalisation.  Runs the GPU plan
    for ``Algorithm.SPLIT_RADIX`` (same kernel as mixed radix).  N = 1 is the
    identity (a copy).
    """
    direction = Direction(direction)
    n = int(signal.shape[-1]) if hasattr(signal, "shape") else len(signal)
    if not is_power_of_two(n):
        raise InvalidLengthError(f"transform length must be a power of two, got {n}")
    if twiddles.n != n:
        raise PlanError(f"twiddle table length {twiddles.n} does not match signal length {n}")
    if verify_twiddles:
        _check_quarter_turns(twiddles.factors)
    precision = "double" if twiddles.factors.dtype == np.complex128 else "single"
    if n == 1:
        x = signal.clone() if hasattr(signal, "clone") else np.array(signal, dtype=twiddles.factors.dtype)
        return x
    from .executor import execute

    plan = make_plan(n, direction, Algorithm.SPLIT_RADIX, precision=precision)
    return execute(plan, signal)
