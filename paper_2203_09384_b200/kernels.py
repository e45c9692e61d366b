"""The reference's ``kernels`` module (kernels.py:28-258) on the GPU.

Two layers, as in the reference:

* the stage-level building blocks -- ``StageBuffer`` and
  ``radix{2,4,8}_stage`` (kernels.py:28-151) keep the reference semantics:
  a buffer of sub-spectra of length ``stride``, one out-of-place
  decimation-in-time stage that multiplies operand (q, j) of each group by
  ``table[(n/span)*q*j mod n]`` (conjugated for the inverse) and combines
  ``radix`` sub-spectra with the same +-1 / +-i / eighth-root arithmetic.
  Each call is one sm_100a kernel over all rows of an ``(N,)`` or
  ``(B, N)`` buffer (``sfft_stage``); ``digit_reverse`` is the matching
  gather (``sfft_permute``).  These exist for custom stage lists;
* the whole-transform entry points -- ``split_radix_transform`` runs the
  plan's fused kernel (both algorithms compute the same DFT: one launch,
  no recursion) and ``count_butterflies`` keeps the reference's arithmetic
  bookkeeping (kernels.py:205-258).

The hot path is ``execute``, which fuses every stage into one pass over HBM.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _native
from .errors import InvalidLengthError, PlanError, ShapeError
from .numerics import TwiddleTable, is_power_of_two
from .planner import Algorithm, Direction, FftPlan, digit_reversal_permutation, make_plan


#: 1/sqrt(2), the radix-8 stage constant (kernels.py:25, :136-141); the GPU
#: kernels use the same value as a compile-time constant (sfft_device.cuh).
SQRT1_2 = float(np.sqrt(0.5))

# ------------------------------------------------------------ stage level
@dataclass
class StageBuffer:
    """``data`` (N,) or (B, N) complex array (numpy or CUDA tensor); ``stride`` =
    length of the sub-spectra entering the next stage (kernels.py:28-38)."""

    data: object
    stride: int


def _torch():
    import torch

    return torch


def _to_device(x, dtype, device=None):
    """``x`` as a contiguous CUDA tensor of ``dtype``: a CUDA tensor stays on
    its device, anything else goes to ``device`` (default: the current one)."""
    torch = _torch()
    want = torch.complex64 if dtype == np.complex64 else torch.complex128
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(device or "cuda")
        return t.to(want).contiguous()
    return torch.from_numpy(np.array(x, dtype=dtype, copy=True)).to(device or "cuda")


def _dtype_of(table: TwiddleTable):
    return np.complex128 if table.factors.dtype == np.complex128 else np.complex64


def _stage(radix: int, buf: StageBuffer, twiddles: TwiddleTable, stage_index: int, direction, out):
    torch = _torch()
    direction = Direction(direction)
    x = buf.data
    n = int(x.shape[-1])
    span = radix * buf.stride
    if buf.stride < 1 or n % span != 0:
        raise PlanError(
            f"stage {stage_index}: radix-{radix} stage needs stride dividing {n}//{radix}, "
            f"got stride {buf.stride} for buffer length {n}"
        )
    if twiddles.n != n:
        raise PlanError(f"stage {stage_index}: twiddle table length {twiddles.n} does not match buffer length {n}")
    dtype = _dtype_of(twiddles)
    is_host = not (isinstance(x, torch.Tensor) and x.is_cuda)
    if out is not None and (tuple(out.shape) != tuple(x.shape)):
        raise PlanError("output buffer must match the stage buffer's shape and dtype")
    xd = _to_device(x, dtype)
    rows = 1 if xd.ndim == 1 else int(xd.shape[0])
    yd = torch.empty_like(xd)
    table = _to_device(twiddles.factors, dtype, xd.device)  # on the buffer's device
    code = _native.SFFT_SINGLE if dtype == np.complex64 else _native.SFFT_DOUBLE
    with torch.cuda.device(xd.device):  # launch on the buffer's device and stream
        stream = torch.cuda.current_stream(xd.device)
        _native.check(
            _native.lib().sfft_stage(
                n, code, radix, buf.stride,
                _native.SFFT_INVERSE if direction is Direction.INVERSE else _native.SFFT_FORWARD,
                ctypes.c_void_p(table.data_ptr()), ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(yd.data_ptr()),
                rows, ctypes.c_void_p(stream.cuda_stream),
            )
        )
    if is_host:
        result = yd.cpu().numpy()
        if out is not None:
            out[...] = result
            result = out
    else:
        result = yd
        if out is not None:
            out.copy_(yd)
            result = out
    return StageBuffer(result, buf.stride * radix)


def radix2_stage(buf, twiddles, stage_index, direction=Direction.FORWARD, out=None) -> StageBuffer:
    """Pairs of sub-spectra: (a, b) -> (a + w b, a - w b)  (kernels.py:83-95)."""
    return _stage(2, buf, twiddles, stage_index, direction, out)


def radix4_stage(buf, twiddles, stage_index, direction=Direction.FORWARD, out=None) -> StageBuffer:
    """4-point DFTs with +-1, +-i only (kernels.py:107-123)."""
    return _stage(4, buf, twiddles, stage_index, direction, out)


def radix8_stage(buf, twiddles, stage_index, direction=Direction.FORWARD, out=None) -> StageBuffer:
    """Two 4-point DFTs plus eighth roots (kernels.py:126-151)."""
    return _stage(8, buf, twiddles, stage_index, direction, out)


RADIX_STAGE = {2: radix2_stage, 4: radix4_stage, 8: radix8_stage}


def digit_reverse(x, stages, precision: str = "single"):
    """``work[..., p] = x[..., perm[p]]`` on the GPU (executor.py:77 with planner.py:62-89)."""
    torch = _torch()
    dtype = np.complex64 if precision == "single" else np.complex128
    xd = _to_device(x, dtype)
    perm = torch.from_numpy(np.array(digit_reversal_permutation(stages), dtype=np.int64)).to(xd.device)
    n = int(xd.shape[-1])
    if perm.numel() != n:
        raise ShapeError(f"stages multiply to {perm.numel()}, signal length is {n}")
    yd = torch.empty_like(xd)
    rows = 1 if xd.ndim == 1 else int(xd.shape[0])
    with torch.cuda.device(xd.device):
        _native.check(
            _native.lib().sfft_permute(
                n, _native.SFFT_SINGLE if dtype == np.complex64 else _native.SFFT_DOUBLE,
                ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(yd.data_ptr()),
                rows, ctypes.c_void_p(torch.cuda.current_stream(xd.device).cuda_stream),
            )
        )
    is_host = not (isinstance(x, torch.Tensor) and x.is_cuda)
    return yd.cpu().numpy() if is_host else yd


# -------------------------------------------------------- whole transform
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
