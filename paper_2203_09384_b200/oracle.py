"""The reference's public ``oracle`` module: direct-summation DFT (oracle.py:18-49).

This is the package API ``stagefft.oracle`` (``dft_matrix`` / ``naive_dft``),
the ground truth the ``verify`` CLI route and ``stats`` compare against -- not
the repository's test oracle under ``/oracle`` (a numpy restatement of the
reference engine that only the tests import).

The O(N^2) sum runs on the GPU as a complex128 matrix product: one ZGEMV for
a signal, one ZGEMM for a whole ``(B, N)`` batch (:func:`naive_dft_batch`,
new).  As in the reference, the phase index ``k*m`` is reduced mod N in
integers before the exponential, accumulation is complex128 and the result
is rounded once.  It never shares code with the FFT kernels.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import CudaError, DomainError, InvalidLengthError, ShapeError
from .planner import Direction
from .validation import COMPLEX_DTYPE, as_signal


def _cuda_torch():
    import torch

    if not torch.cuda.is_available():
        raise CudaError("the direct DFT runs on the GPU; no CUDA device is visible")
    return torch


def _phase_angles(n: int, direction, device):
    """Angles sign*2*pi*((k*m) mod n)/n as a float64 (n, n) tensor on ``device``."""
    torch = _cuda_torch()
    k = torch.arange(n, dtype=torch.int64, device=device)
    reduced = (k[:, None] * k[None, :]).remainder_(n)
    sign = 1.0 if Direction(direction) is Direction.INVERSE else -1.0
    return reduced.to(torch.float64).mul_(sign * 2.0 * math.pi / n)


def _fourier_matrix(n: int, direction, device):
    torch = _cuda_torch()
    ang = _phase_angles(n, direction, device)
    return torch.complex(torch.cos(ang), torch.sin(ang))


def dft_matrix(n: int, direction: Direction = Direction.FORWARD) -> np.ndarray:
    """The n x n Fourier matrix, complex128, entry (k, m) = exp(-+2 pi i (k m mod n) / n).

    Returned as a host numpy array like the reference (oracle.py:18-30);
    computed on the GPU.
    """
    n = int(n)
    if n < 1:
        raise InvalidLengthError(f"transform length must be >= 1, got {n}")
    return _fourier_matrix(n, direction, "cuda").cpu().numpy()


def naive_dft(signal, direction: Direction = Direction.FORWARD) -> np.ndarray:
    """Direct DFT of one 1-D signal of any positive length (oracle.py:33-49).

    The input is validated and rounded to complex64 first (``as_signal``),
    summed in complex128 on the GPU, divided by n for the inverse, and
    rounded to complex64 once.  The input is never modified.
    """
    x = as_signal(signal)
    direction = Direction(direction)
    torch = _cuda_torch()
    n = x.shape[0]
    xd = torch.from_numpy(x.astype(np.complex128)).cuda()
    y = _fourier_matrix(n, direction, xd.device) @ xd
    if direction is Direction.INVERSE:
        y = y / n
    return y.to(torch.complex64).cpu().numpy()


def naive_dft_batch(X, direction: Direction = Direction.FORWARD, *, precision: str = "single"):
    """Direct DFT of every row of a ``(B, N)`` batch: one ZGEMM.

    ``precision`` "single" rounds the input to complex64 first and the
    result to complex64 at the end (the reference's convention per row);
    "double" keeps complex128 throughout.  A CUDA tensor stays on its device
    and a tensor comes back as a tensor; numpy comes back as numpy.
    """
    torch = _cuda_torch()
    direction = Direction(direction)
    is_tensor = isinstance(X, torch.Tensor)
    t = X if is_tensor else torch.from_numpy(np.ascontiguousarray(X))
    if t.ndim != 2 or 0 in t.shape:
        raise ShapeError(f"expected a non-empty (B, N) batch, got shape {tuple(t.shape)}")
    if t.dtype == torch.bool:
        raise DomainError(f"batch has non-numeric dtype {t.dtype}")
    dev = t.device if t.is_cuda else torch.device("cuda")
    single = precision == "single"
    x = t.to(dev).to(torch.complex64 if single else torch.complex128)
    if not bool(torch.isfinite(torch.view_as_real(x)).all()):
        raise DomainError("batch contains NaN or Inf values")
    n = x.shape[1]
    y = x.to(torch.complex128) @ _fourier_matrix(n, direction, dev).T
    if direction is Direction.INVERSE:
        y = y / n
    if single:
        y = y.to(torch.complex64)
    if is_tensor:
        return y if t.is_cuda else y.cpu()
    return y.cpu().numpy()


__all__ = ["COMPLEX_DTYPE", "dft_matrix", "naive_dft", "naive_dft_batch"]
