"""Synthetic inputs (mirror of signalgen.py:14-41) plus a batched generator.

``generate_batch(B, N, seed)`` draws ``Philox(key=seed).uniform(-1, 1,
size=(2, B, N))`` -- the reference draw order with a batch axis -- so row 0
of a B=1 batch equals ``generate("random", N, seed)`` bit for bit.
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidLengthError

KINDS = ("ramp", "impulse", "constant", "random")
_DTYPES = {"single": np.complex64, "double": np.complex128}


def generate(kind: str, n: int, seed: int = 0, precision: str = "single") -> np.ndarray:
    """One length-n test signal: ramp (k, 0), impulse, constant or random."""
    if n < 1:
        raise InvalidLengthError(f"signal length must be >= 1, got {n}")
    dtype = _DTYPES[precision]
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
        return generate_batch(1, n, seed, precision)[0]
    raise ValueError(f"unknown signal kind {kind!r}; expected one of {KINDS}")


def generate_batch(batch: int, n: int, seed: int = 0, precision: str = "single", out=None) -> np.ndarray:
    """(batch, n) Philox-uniform complex rows; ``out`` may be a preallocated
    (e.g. pinned) array of the right shape and dtype to fill in place."""
    if n < 1 or batch < 1:
        raise InvalidLengthError(f"batch and length must be >= 1, got ({batch}, {n})")
    dtype = _DTYPES[precision]
    rng = np.random.Generator(np.random.Philox(key=seed))
    parts = rng.uniform(-1.0, 1.0, size=(2, batch, n))
    if out is None:
        return (parts[0] + 1j * parts[1]).astype(dtype)
    view = out.view(np.float32 if dtype == np.complex64 else np.float64).reshape(batch, n, 2)
    view[..., 0] = parts[0]
    view[..., 1] = parts[1]
    return out
