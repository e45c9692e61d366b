"""Exception tree of the reference (errors.py:9-34), plus a CUDA failure class.

Each C-ABI status code (include/sfft.h) maps onto exactly one class here, so
callers of the GPU path catch the same types as callers of the reference.
"""


class FftError(Exception):
    """Root of every error raised by this package (errors.py:9-10)."""


class InvalidLengthError(FftError, ValueError):
    """Length is empty, non-positive or not a power of two (errors.py:13-14)."""


class UnsupportedLengthError(InvalidLengthError):
    """Power of two outside the engine range (errors.py:17-18)."""


class PlanError(FftError, ValueError):
    """Inconsistent stage list / radix / kernel variant (errors.py:21-22)."""


class ShapeError(FftError, ValueError):
    """Array arguments disagree in shape or dimensionality (errors.py:25-26)."""


class DomainError(FftError, ValueError):
    """NaN/Inf or non-numeric input (errors.py:29-30)."""


class InsufficientDataError(FftError, ValueError):
    """Kept for API parity with the reference tree (errors.py:33-34)."""


class CudaError(FftError, RuntimeError):
    """The device or CUDA runtime failed (no reference analogue)."""


class ArgumentError(FftError, ValueError):
    """Null/misaligned buffer or bad enum passed across the C ABI."""


#: C-ABI status code -> exception class (include/sfft.h SFFT_ERR_*)
STATUS_TO_ERROR = {
    1: InvalidLengthError,
    2: UnsupportedLengthError,
    3: PlanError,
    4: ShapeError,
    5: DomainError,
    6: CudaError,
    7: ArgumentError,
}
