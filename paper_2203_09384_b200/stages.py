"""The reference's stage-level API on the GPU (kernels.py:28-151).

``StageBuffer`` and ``radix{2,4,8}_stage`` keep the reference semantics -- a
buffer of sub-spectra of length ``stride``, one out-of-place
decimation-in-time stage that multiplies operand (q, j) of each group by
``table[(n/span)*q*j mod n]`` (conjugated for the inverse) and combines
``radix`` sub-spectra with the same +-1 / +-i / eighth-root arithmetic --
but each call is one sm_100a kernel over all rows of a ``(N,)`` or ``(B, N)``
buffer (``sfft_stage``), and ``digit_reverse`` is the matching gather
(``sfft_permute``).

This is the building-block API for custom stage lists; the hot path is
``execute``, which fuses every stage into one pass over HBM.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import PlanError, ShapeError
from .numerics import TwiddleTable
from .planner import Direction, digit_reversal_permutation


@dataclass
class StageBuffer:
    """``data`` (N,) or (B, N) complex array (numpy or CUDA tensor); ``stride`` =
    length of the sub-spectra entering the next stage (kernels.py:28-38)."""

    data: object
    stride: int


def _torch():
    import torch

    return torch


def _to_device(x, dtype):
    torch = _torch()
    want = torch.complex64 if dtype == np.complex64 else torch.complex128
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
        return t.to(want).contiguous()
    return torch.from_numpy(np.array(x, dtype=dtype, copy=True)).cuda()


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
    table = _to_device(twiddles.factors, dtype)
    code = _native.SFFT_SINGLE if dtype == np.complex64 else _native.SFFT_DOUBLE
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
    perm = torch.from_numpy(np.array(digit_reversal_permutation(stages), dtype=np.int64)).cuda()
    xd = _to_device(x, dtype)
    n = int(xd.shape[-1])
    if perm.numel() != n:
        raise ShapeError(f"stages multiply to {perm.numel()}, signal length is {n}")
    yd = torch.empty_like(xd)
    rows = 1 if xd.ndim == 1 else int(xd.shape[0])
    _native.check(
        _native.lib().sfft_permute(
            n, _native.SFFT_SINGLE if dtype == np.complex64 else _native.SFFT_DOUBLE,
            ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(yd.data_ptr()),
            rows, ctypes.c_void_p(torch.cuda.current_stream(xd.device).cuda_stream),
        )
    )
    is_host = not (isinstance(x, torch.Tensor) and x.is_cuda)
    return yd.cpu().numpy() if is_host else yd
