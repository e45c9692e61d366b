"""Plan construction (mirror of planner.py:1-188) with precision and batch axes.

``make_plan`` keeps the reference signature and adds three keyword-only
arguments: ``precision`` ("single" | "double"), ``batch`` (rows per execute,
``None`` = any) and ``device`` (CUDA ordinal, ``None`` = the input's device).

The reference-facing fields (``stages``, ``permutation``, ``twiddles``,
``scale``, ``chunk``) are computed exactly as the reference computes them, so
code that inspects a plan keeps working.  The GPU itself does not use the
digit-reversal permutation: its Stockham schedule sorts in flight, and the
native plan (created per device on first use, ``sfft_plan_create``) picks its
own radix-8/16 pass schedule, reported by :meth:`FftPlan.kernel_info`.

Deviations from the reference, all deliberate:
* supported lengths are 2..2048 (the reference engine starts at 8,
  planner.py:21); N = 2 and 4 were reachable only through the split-radix
  recursion there;
* ``Algorithm.SPLIT_RADIX`` is accepted and reported, but both algorithms run
  the same GPU kernel (they compute the same DFT; the split recursion is a
  CPU scheduling choice).
"""

from __future__ import annotations

import ctypes
import math
import threading
import weakref
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native
from .errors import InvalidLengthError, PlanError, ShapeError, UnsupportedLengthError
from .numerics import TwiddleTable, build_twiddle_table, is_power_of_two

ENGINE_MIN_LENGTH = 2
ENGINE_MAX_LENGTH = 2048
SUPPORTED_RADICES = (2, 4, 8)
#: Transform lengths the GPU engine accepts: 2**1 .. 2**11.
SUPPORTED_LENGTHS = tuple(2**p for p in range(1, 12))


class Direction(Enum):
    FORWARD = "forward"
    INVERSE = "inverse"


class Algorithm(Enum):
    MIXED_RADIX = "mixed"
    SPLIT_RADIX = "split"


class Precision(Enum):
    SINGLE = "single"  # complex64, the reference engine dtype
    DOUBLE = "double"  # complex128

    @property
    def dtype(self):
        return np.complex64 if self is Precision.SINGLE else np.complex128

    @property
    def code(self) -> int:
        return _native.SFFT_SINGLE if self is Precision.SINGLE else _native.SFFT_DOUBLE


def factorize_stages(n: int) -> list[int]:
    """Greedy radix-8-first factorisation (planner.py:38-59), range 2..2048."""
    if not is_power_of_two(n):
        raise InvalidLengthError(f"transform length must be a power of two, got {n}")
    if not ENGINE_MIN_LENGTH <= n <= ENGINE_MAX_LENGTH:
        raise UnsupportedLengthError(
            f"length {n} outside supported range [{ENGINE_MIN_LENGTH}, {ENGINE_MAX_LENGTH}]"
        )
    stages = []
    rest = n
    while rest % 8 == 0:
        stages.append(8)
        rest //= 8
    if rest > 1:
        stages.append(rest)
    return stages


def digit_reversal_permutation(stages) -> np.ndarray:
    """Input order of an in-place DIT pass over ``stages`` (planner.py:62-89).

    ``work[p] = x[perm[p]]``; digits of p are read with the last stage most
    significant and reversed.  Computed for all indices at once.
    """
    radices = [int(r) for r in stages]
    if not radices:
        raise PlanError("stage list is empty")
    for r in radices:
        if r not in SUPPORTED_RADICES:
            raise PlanError(f"unsupported radix {r}; expected one of {SUPPORTED_RADICES}")
    n = math.prod(radices)
    rem = np.arange(n, dtype=np.int64)
    src = np.zeros(n, dtype=np.int64)
    weight, mult = n, 1
    for r in reversed(radices):
        weight //= r
        digit, rem = np.divmod(rem, weight)
        src += digit * mult
        mult *= r
    perm = src.astype(np.intp)
    perm.setflags(write=False)
    return perm


class _NativePlans:
    """Per-device native plan handles, created on first use, freed with the plan."""

    def __init__(self, spec):
        self.spec = spec  # (n, precision code, direction code, batch, variant)
        self.handles: dict[int, int] = {}
        self.real_input: dict[int, bool] = {}  # device -> kernel has the real-input loader
        self.lock = threading.Lock()
        self._finalizer = weakref.finalize(self, _NativePlans._destroy, self.handles)

    @staticmethod
    def _destroy(handles):
        if not handles:
            return
        lib = _native.lib()
        for h in handles.values():
            lib.sfft_plan_destroy(ctypes.c_void_p(h))
        handles.clear()

    def handle(self, device: int) -> int:
        h = self.handles.get(device)
        if h is None:
            with self.lock:
                h = self.handles.get(device)
                if h is None:
                    n, prec, direc, batch, variant = self.spec
                    out = ctypes.c_void_p()
                    _native.check(
                        _native.lib().sfft_plan_create_variant(
                            ctypes.byref(out), n, prec, direc, batch, device, variant
                        )
                    )
                    h = out.value
                    self.handles[device] = h
        return h  # the C-ABI argtypes (c_void_p) take the address as an int


@dataclass(frozen=True)
class FftPlan:
    """Immutable recipe for one length/direction/algorithm/precision.

    Fields up to ``chunk`` are the reference's (planner.py:92-136); ``chunk``
    stays ``length`` because a GPU launch always runs whole transforms.
    Equality and hashing follow the reference (arrays excluded) and include
    the new ``precision`` and ``batch`` axes.
    """

    length: int
    direction: Direction
    algorithm: Algorithm
    stages: tuple[int, ...]
    permutation: np.ndarray
    twiddles: TwiddleTable
    scale: float
    chunk: int
    precision: Precision = Precision.SINGLE
    batch: int | None = None
    device: int | None = None
    variant: int = 0
    _handles: _NativePlans = field(init=False, repr=False, compare=False, default=None)

    def __post_init__(self):
        spec = (
            self.length,
            self.precision.code,
            _native.SFFT_INVERSE if self.direction is Direction.INVERSE else _native.SFFT_FORWARD,
            int(self.batch or 0),
            int(self.variant),
        )
        object.__setattr__(self, "_handles", _NativePlans(spec))

    def __eq__(self, other) -> bool:
        if not isinstance(other, FftPlan):
            return NotImplemented
        return (
            self.length == other.length
            and self.direction is other.direction
            and self.algorithm is other.algorithm
            and self.stages == other.stages
            and self.scale == other.scale
            and self.chunk == other.chunk
            and self.precision is other.precision
            and self.batch == other.batch
        )

    def __hash__(self) -> int:
        return hash(
            (self.length, self.direction, self.algorithm, self.stages, self.scale, self.precision)
        )

    @property
    def dtype(self):
        return self.precision.dtype

    def supports_real_input(self, device: int) -> bool:
        """Whether the kernel reads real rows directly (sfft_execute_ex, SFFT_INPUT_REAL)."""
        cache = self._handles.real_input
        ok = cache.get(device)
        if ok is None:
            ok = cache[device] = bool(self.kernel_info(device)["real_input"])
        return ok

    def native_handle(self, device: int) -> int:
        """The per-device ``sfft_plan_t`` (created and uploaded on first call)."""
        return self._handles.handle(int(device))

    def kernel_info(self, device: int = 0) -> dict:
        """GPU schedule of this plan on ``device`` (sfft_plan_info)."""
        info = _native.PlanInfo()
        _native.check(_native.lib().sfft_plan_info(self.native_handle(device), ctypes.byref(info)))
        return info.as_dict()


def make_plan(
    length: int,
    direction: Direction = Direction.FORWARD,
    algorithm: Algorithm = Algorithm.MIXED_RADIX,
    *,
    stages=None,
    precision: Precision | str = Precision.SINGLE,
    batch: int | None = None,
    device: int | None = None,
    variant: int = 0,
) -> FftPlan:
    """Build the plan for one transform shape (planner.py:139-188).

    Strings are accepted for the enums.  ``stages`` overrides the greedy
    factorisation exactly as in the reference (validated, recorded, and used
    for ``permutation``); the GPU schedule is chosen by the native planner.
    No device memory is touched here: the per-device native plan is created
    on the first execute on that device.
    """
    direction = Direction(direction)
    algorithm = Algorithm(algorithm)
    precision = Precision(precision)
    default_stages = factorize_stages(length)  # validates length
    if stages is None:
        stage_tuple = tuple(default_stages)
    else:
        stage_tuple = tuple(int(r) for r in stages)
        for r in stage_tuple:
            if r not in SUPPORTED_RADICES:
                raise PlanError(f"unsupported radix {r}; expected one of {SUPPORTED_RADICES}")
        if math.prod(stage_tuple) != length:
            raise PlanError(
                f"stages {stage_tuple} multiply to {math.prod(stage_tuple)}, not {length}"
            )
    if batch is not None:
        batch = int(batch)
        if batch < 1:
            raise ShapeError(f"batch must be a positive row count, got {batch}")
    nvar = _native.lib().sfft_num_variants(length, precision.code)
    if not 0 <= int(variant) < nvar:
        raise PlanError(f"kernel variant {variant} does not exist (n={length}: {nvar} variants)")
    if algorithm is Algorithm.SPLIT_RADIX:
        permutation = np.arange(length, dtype=np.intp)
        permutation.setflags(write=False)
    else:
        permutation = digit_reversal_permutation(stage_tuple)
    return FftPlan(
        length=length,
        direction=direction,
        algorithm=algorithm,
        stages=stage_tuple,
        permutation=permutation,
        twiddles=build_twiddle_table(length, precision.value),
        scale=1.0 / length if direction is Direction.INVERSE else 1.0,
        chunk=length,
        precision=precision,
        batch=batch,
        device=None if device is None else int(device),
        variant=int(variant),
    )
