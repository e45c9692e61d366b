"""Batched plan execution on the GPU (mirror of executor.py:1-96).

``execute(plan, signal)`` keeps the reference contract -- the input is never
written, the output is fresh memory, repeated runs are bit-identical, one plan
may be shared by many threads -- and widens it:

* ``signal`` may be 1-D ``(N,)`` (reference behaviour) or batched ``(B, N)``;
  anything else, or a last axis != plan length, is a ``ShapeError``
  (executor.py:64-69);
* numpy / array-like input runs through the native host pipeline
  (``sfft_execute_host``: chunked H2D -> kernel -> D2H) and returns numpy;
  a torch CUDA tensor stays on its device (``sfft_execute_sync`` on the
  current stream) and returns a tensor there; ``launch`` is the raw
  asynchronous entry (``sfft_execute``) for pipelines that sync themselves.

Every path launches the sm_100a kernels; there is no CPU fallback.  NaN/Inf
input raises ``DomainError`` (executor.py:72-73) -- detected inside the kernel
while it loads the data, so validation costs no extra pass over memory.
"""

from __future__ import annotations

import ctypes
import math
import mmap
import time
from typing import NamedTuple

import numpy as np

from . import _native
from .errors import DomainError, ShapeError
from .planner import FftPlan
from .validation import check_batch

try:  # torch is the device-memory/stream plumbing; numpy input works without it
    import torch
except ImportError:  # pragma: no cover - torch is in the image
    torch = None


class TimedExecution(NamedTuple):
    """executor.py:28-31: output plus host dispatch and device compute time."""

    output: object
    dispatch_us: float
    compute_us: float


def _is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _raw_stream(device_index: int) -> int:
    """cudaStream_t of torch's current stream on a device.

    torch.cuda.current_stream() builds a Stream object (~2.3 us per call on
    the B200 host, a sixth of a small execute()); the raw getter behind it
    returns the handle directly."""
    return _get_raw_stream(device_index)


def _get_raw_stream_slow(device_index: int) -> int:
    return torch.cuda.current_stream(device_index).cuda_stream


_get_raw_stream = getattr(getattr(torch, "_C", None), "_cuda_getCurrentRawStream", None) or _get_raw_stream_slow


_cuda_seen = False  # torch.cuda.is_available() costs ~2 us; once True it stays True


def _default_device(plan: FftPlan) -> int:
    global _cuda_seen
    if plan.device is not None:
        return plan.device
    if torch is not None and (_cuda_seen or torch.cuda.is_available()):
        _cuda_seen = True
        return torch.cuda.current_device()
    return 0


def _addr(a: np.ndarray) -> int:
    """Data address of a C-contiguous array: the buffer protocol (~0.6 us)
    instead of ``a.ctypes.data`` (~2 us, a fresh ctypes helper object per
    access); read-only arrays take the slow route."""
    try:
        return ctypes.addressof(ctypes.c_char.from_buffer(a))
    except (TypeError, ValueError, BufferError):
        return a.ctypes.data


# ----------------------------------------------------------------- numpy path
def _prepare_host(plan: FftPlan, signal, allow_real: bool = False):
    """(original array, contiguous input for the kernel, rows, input kind).

    With ``allow_real``, real input whose plan kernel has the real loader is
    passed as real rows of the plan's real type (half the H2D bytes);
    otherwise it is widened to the plan dtype here, as validation.py:26 /
    executor.py:74 do (complex128 -> complex64 for a single-precision plan).
    """
    x = np.asarray(signal)
    rows = check_batch(plan.length, x.shape, plan.batch)
    if x.dtype.kind not in "fciu":
        raise DomainError(f"signal has non-numeric dtype {x.dtype}")
    if allow_real and x.dtype.kind != "c" and plan.supports_real_input(_default_device(plan)):
        real_t = np.float32 if plan.dtype == np.complex64 else np.float64
        return x, np.ascontiguousarray(x, dtype=real_t), rows, _native.SFFT_INPUT_REAL
    xc = np.ascontiguousarray(x, dtype=plan.dtype)
    if _addr(xc) % 16:
        xc = xc.copy()
    return x, xc, rows, _native.SFFT_INPUT_COMPLEX


_HUGE_OUTPUT_BYTES = 32 << 20


def _empty_host(shape, dtype) -> np.ndarray:
    """Output array for the host path.

    Large outputs come from an anonymous mapping advised for transparent huge
    pages: the pipeline's drain copies first-touch every page, and 2 MiB
    pages cut that fault cost -- 36.8 -> 31.4 ms for a 512 MiB fresh output
    on the B200 host (tools/thp_probe.py).  Small ones use np.empty."""
    nbytes = math.prod(shape) * np.dtype(dtype).itemsize
    if nbytes < _HUGE_OUTPUT_BYTES or not hasattr(mmap, "MADV_HUGEPAGE"):
        return np.empty(shape, dtype=dtype)
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    try:
        m.madvise(mmap.MADV_HUGEPAGE)
    except OSError:  # THP disabled: still a valid (4 KiB-paged) buffer
        pass
    return np.frombuffer(m, dtype=dtype).reshape(shape)


def _execute_host(plan: FftPlan, signal, out=None, timed: bool = False):
    """numpy path; with ``timed``, returns (out, dispatch_us, compute_us) where
    dispatch covers validation and conversion and compute the native call
    (H2D copies, kernels and D2H copies of the host pipeline)."""
    t0 = time.perf_counter_ns()
    x, xc, rows, kind = _prepare_host(plan, signal, allow_real=True)
    if out is None:
        out = _empty_host(xc.shape, plan.dtype)
    elif (
        not isinstance(out, np.ndarray)
        or out.dtype != plan.dtype
        or out.size != xc.size
        or not out.flags.c_contiguous
        or _addr(out) % 16
    ):
        raise ShapeError("out must be a C-contiguous, 16-byte aligned array of the plan dtype and size")
    handle = plan.native_handle(_default_device(plan))
    t1 = time.perf_counter_ns()
    _native.check(_native.lib().sfft_execute_host_ex(handle, _addr(xc), _addr(out), rows, kind))
    if not timed:
        return out
    t2 = time.perf_counter_ns()
    return out, (t1 - t0) / 1000.0, (t2 - t1) / 1000.0


# ----------------------------------------------------------------- torch path
def _prepare_device(plan: FftPlan, x):
    """(input tensor for the kernel, rows, input kind).

    Real input (executor.py:74 casts it to complex; test_executor.py:89-92)
    goes to the kernel as real rows when its loader supports that: it reads
    half the bytes and zeroes the imaginary parts in registers, instead of a
    widening pass to complex first."""
    rows = check_batch(plan.length, x.shape, plan.batch)
    if x.dtype == torch.bool:  # numpy kind "b" is rejected too (executor.py:70-71)
        raise DomainError(f"signal has non-numeric dtype {x.dtype}")
    single = plan.dtype == np.complex64
    if not x.is_complex() and plan.supports_real_input(x.get_device()):
        xr = x.to(torch.float32 if single else torch.float64).contiguous()
        if xr.data_ptr() % 16:  # the real loaders read 16-byte chunks (sfft.h)
            xr = xr.clone()
        return xr, rows, _native.SFFT_INPUT_REAL
    xc = x.to(torch.complex64 if single else torch.complex128).contiguous()
    if xc.data_ptr() % 16:
        xc = xc.clone()
    return xc, rows, _native.SFFT_INPUT_COMPLEX


def launch(plan: FftPlan, x_in, x_out, rows: int, *, stream=None, flag=None) -> None:
    """Asynchronous launch on device tensors (no validation, no sync).

    ``x_in``/``x_out`` are contiguous CUDA tensors holding ``rows``
    sequences: ``x_out`` of the plan dtype, ``x_in`` of the plan dtype or of
    its real type (float32 / float64 rows, read by the real-input loader);
    ``flag`` an int32 CUDA tensor the kernel ORs 1 into on NaN/Inf input.
    Kernels are launched with programmatic dependent launch, so back-to-back
    calls overlap one launch's ramp with the previous one's drain while
    staying ordered.  This is the call ``bench.py`` times.
    """
    dev = x_in.get_device()
    raw = _raw_stream(dev) if stream is None else stream.cuda_stream
    kind = _native.SFFT_INPUT_COMPLEX if x_in.is_complex() else _native.SFFT_INPUT_REAL
    _native.check(
        _native.lib().sfft_execute_ex(
            plan.native_handle(dev),
            x_in.data_ptr(),
            x_out.data_ptr(),
            rows,
            raw,
            None if flag is None else flag.data_ptr(),
            kind,
        )
    )


def _execute_device(plan: FftPlan, x, timed: bool = False, out=None):
    t0 = time.perf_counter_ns()
    xc, rows, kind = _prepare_device(plan, x)
    cdt = torch.complex64 if plan.dtype == np.complex64 else torch.complex128
    if out is None:
        out = torch.empty(xc.shape, dtype=cdt, device=xc.device)
    elif (
        not _is_torch(out)
        or out.device != xc.device
        or out.dtype != cdt
        or out.numel() != xc.numel()
        or not out.is_contiguous()
        or out.data_ptr() % 16
    ):
        raise ShapeError("out must be a contiguous, 16-byte aligned tensor of the plan dtype on the input device")
    dev = xc.get_device()
    handle = plan.native_handle(dev)
    kernel_ms = ctypes.c_float(0.0) if timed else None
    t1 = time.perf_counter_ns()
    # one C call: launch, wait, read the mapped NaN/Inf flag (DomainError)
    _native.check(
        _native.lib().sfft_execute_sync_ex(
            handle,
            xc.data_ptr(),
            out.data_ptr(),
            rows,
            _raw_stream(dev),
            ctypes.byref(kernel_ms) if timed else None,
            kind,
        )
    )
    return out, (t1 - t0) / 1000.0, kernel_ms.value * 1000.0 if timed else 0.0


# ----------------------------------------------------------------- public API
def execute(plan: FftPlan, signal, *, out=None):
    """Run ``plan`` on ``signal`` and return fresh output (executor.py:50-52).

    ``out`` (optional, not in the reference) receives the result instead of a
    fresh allocation -- e.g. a pinned host array, so the D2H copy runs at full
    DMA rate.  It must not alias ``signal`` unless in-place is intended.
    """
    if _is_torch(signal):
        if signal.is_cuda:
            return _execute_device(plan, signal, out=out)[0]
        return torch.from_numpy(_execute_host(plan, signal.numpy(), None if out is None else out.numpy()))
    return _execute_host(plan, signal, out)


def execute_timed(plan: FftPlan, signal) -> TimedExecution:
    """execute plus timing (executor.py:55-96).

    ``dispatch_us``: host time from entry to the native call (validation,
    dtype conversion, output allocation).  ``compute_us``: for a CUDA tensor,
    the kernel's device time from CUDA events recorded around the launch on
    its stream (sfft_execute_sync); for host input, the whole native host
    pipeline -- H2D copies, kernels and D2H copies -- as the reference's
    compute phase covers everything after the permute.
    """
    if _is_torch(signal):
        if signal.is_cuda:
            return TimedExecution(*_execute_device(plan, signal, timed=True))
        out, dispatch_us, compute_us = _execute_host(plan, signal.numpy(), timed=True)
        return TimedExecution(torch.from_numpy(out), dispatch_us, compute_us)
    return TimedExecution(*_execute_host(plan, signal, timed=True))
