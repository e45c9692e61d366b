"""Boundary checks of the reference's ``validation`` module (validation.py:10-57).

The reference funnels every entry point through three helpers that coerce
host arrays to complex64 and scan them for NaN/Inf.  This package keeps the
names, the exception classes and their order of precedence (shape, then
emptiness, then dtype, then finiteness), and changes three things:

* the target dtype is a parameter -- a double-precision plan validates to
  complex128 instead of silently downcasting (validation.py:26 always casts
  to complex64);
* CUDA tensors are accepted and stay on their device: only their shape and
  dtype are checked here, because the FFT kernels fuse the NaN/Inf scan into
  their single pass over HBM (``sfft_execute_sync`` -> ``DomainError``);
* :func:`check_batch` is the executor's shape rule for the widened
  ``(N,)`` / ``(B, N)`` input (executor.py:64-69 for the 1-D case).
"""

from __future__ import annotations

import numpy as np

from .errors import DomainError, InvalidLengthError, ShapeError

#: The reference engine's sample dtype (validation.py:10); single-precision
#: plans keep it, double-precision plans use complex128.
COMPLEX_DTYPE = np.complex64

_NUMERIC_KINDS = frozenset("fciu")


def _torch_tensor(x):
    """``x`` if it is a torch tensor, else None (torch is optional here)."""
    try:
        import torch
    except ImportError:  # pragma: no cover - torch is in the image
        return None
    return x if isinstance(x, torch.Tensor) else None


def _torch_bool():
    import torch

    return torch.bool


def _screen(arr: np.ndarray, name: str, dtype) -> np.ndarray:
    """dtype kind -> cast -> finiteness, the tail every helper shares."""
    if arr.dtype.kind not in _NUMERIC_KINDS:
        raise DomainError(f"{name} has non-numeric dtype {arr.dtype}")
    cast = arr.astype(dtype, copy=False)
    if not np.isfinite(cast).all():  # complex: finite iff both parts are
        raise DomainError(f"{name} contains NaN or Inf values")
    return cast


def as_signal(values, *, name: str = "signal", dtype=COMPLEX_DTYPE) -> np.ndarray:
    """One 1-D, non-empty, numeric, finite signal as ``dtype`` (validation.py:13-30).

    An array already of ``dtype`` is returned without a copy: treat the
    result as read-only.
    """
    arr = np.asarray(values)
    if arr.ndim != 1:
        raise ShapeError(f"{name} must be one-dimensional, got shape {arr.shape}")
    if arr.shape[0] == 0:
        raise InvalidLengthError(f"{name} is empty")
    return _screen(arr, name, dtype)


def check_same_length(a, b, *, names=("lhs", "rhs")) -> None:
    """ShapeError unless two 1-D signals have the same length (validation.py:33-38)."""
    la, lb = int(a.shape[0]), int(b.shape[0])
    if la != lb:
        raise ShapeError(f"{names[0]} and {names[1]} lengths differ: {la} vs {lb}")


def check_signal_matrix(X, *, name: str = "X", dtype=COMPLEX_DTYPE, kernel_checks: bool = False):
    """A 2-D batch with one signal per row (validation.py:40-57).

    By default numpy input is cast to ``dtype`` and scanned for NaN/Inf, as
    the reference does.  With ``kernel_checks`` (the estimator's GPU route)
    the value checks are left to the FFT kernel, which ORs a NaN/Inf flag
    while it loads the rows (-> the same ``DomainError``): real rows stay
    real for the kernel's real-input loader (half the bytes, no widening
    pass) and nothing is scanned on the host.  A torch tensor is returned as
    is after the shape and dtype checks.
    """
    t = _torch_tensor(X)
    shape = tuple(X.shape) if t is not None else np.shape(X)
    if len(shape) == 1:
        raise ShapeError(
            f"{name} must be 2-D with one signal per row; reshape a single signal with {name}.reshape(1, -1)"
        )
    if len(shape) != 2:
        raise ShapeError(f"{name} must be 2-D, got shape {shape}")
    if 0 in shape:
        raise InvalidLengthError(f"{name} is empty, shape {shape}")
    if t is not None:
        if t.dtype is _torch_bool():  # numpy kind "b" is rejected too
            raise DomainError(f"{name} has non-numeric dtype {t.dtype}")
        return t
    arr = np.asarray(X)
    if not kernel_checks:
        return _screen(arr, name, dtype)
    if arr.dtype.kind not in _NUMERIC_KINDS:
        raise DomainError(f"{name} has non-numeric dtype {arr.dtype}")
    return arr.astype(dtype, copy=False) if arr.dtype.kind == "c" else arr


def check_batch(length: int, shape, batch: int | None = None) -> int:
    """Rows of an ``(N,)`` or ``(B, N)`` input for a length-``length`` plan.

    executor.py:64-69 requires 1-D input of the plan length; the batched
    path also takes 2-D input, whose last axis is the transform axis (so a
    ``(8, 8)`` matrix fed to a length-64 plan is still a ShapeError, as
    tests/test_executor.py:95-100 expects).  ``batch`` is the plan's
    optional fixed row count.
    """
    ndim = len(shape)  # hot path of every execute(): plain indexing, no conversions
    if ndim != 1 and ndim != 2:
        raise ShapeError(f"signal must be (N,) or (batch, N), got shape {tuple(shape)}")
    if shape[-1] != length:
        raise ShapeError(f"signal length {shape[-1]} does not match plan length {length}")
    if ndim == 1:
        return 1
    rows = int(shape[0])
    if rows == 0:
        raise InvalidLengthError(f"signal batch is empty, shape {tuple(shape)}")
    if batch is not None and rows != batch:
        raise ShapeError(f"signal has {rows} rows; the plan was made for batch={batch}")
    return rows
