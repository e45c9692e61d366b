"""ctypes binding of the C ABI in include/sfft.h.

The shared library is built in-tree (``paper_2203_09384_b200/_lib/libsfft.so``,
see ``build.py``).  There is deliberately no fallback: if the library is
missing, importing the execution path raises, so a GPU run can never pass on a
CPU or eager-PyTorch substitute.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import STATUS_TO_ERROR, FftError

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libsfft.so")

SFFT_SINGLE, SFFT_DOUBLE = 0, 1
SFFT_FORWARD, SFFT_INVERSE = 0, 1
SFFT_KERNEL_STOCKHAM, SFFT_KERNEL_TILE, SFFT_KERNEL_SPLIT2, SFFT_KERNEL_FOURSTEP = 0, 1, 2, 3
SFFT_INPUT_COMPLEX, SFFT_INPUT_REAL = 0, 1

#: every symbol include/sfft.h declares (tests check the .so exports them all)
EXPORTED_SYMBOLS = (
    "sfft_version",
    "sfft_num_variants",
    "sfft_build_twiddle_table",
    "sfft_plan_create",
    "sfft_plan_create_variant",
    "sfft_plan_destroy",
    "sfft_plan_info",
    "sfft_variant_info",
    "sfft_plan_twiddles",
    "sfft_execute",
    "sfft_execute_sync",
    "sfft_execute_ex",
    "sfft_execute_sync_ex",
    "sfft_execute_host",
    "sfft_execute_host_ex",
    "sfft_permute",
    "sfft_stage",
    "sfft_last_error",
)


class PlanInfo(ctypes.Structure):
    """Mirror of sfft_plan_info_t."""

    _fields_ = [
        ("n", ctypes.c_int32),
        ("precision", ctypes.c_int32),
        ("direction", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("batch", ctypes.c_int64),
        ("kernel", ctypes.c_int32),
        ("elems_per_thread", ctypes.c_int32),
        ("seqs_per_cta", ctypes.c_int32),
        ("threads_per_cta", ctypes.c_int32),
        ("smem_bytes", ctypes.c_int32),
        ("num_passes", ctypes.c_int32),
        ("radices", ctypes.c_int32 * 8),
        ("twiddle_elems", ctypes.c_int64),
        ("variant", ctypes.c_int32),
        ("layout", ctypes.c_int32),
        ("twiddle_policy", ctypes.c_int32),
        ("loader", ctypes.c_int32),
        ("smem_carveout", ctypes.c_int32),
        ("pipeline_stages", ctypes.c_int32),
        ("real_input", ctypes.c_int32),
        ("real_loader", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_ if name != "reserved"}
        d["radices"] = [int(r) for r in self.radices[: self.num_passes]]
        return d


_lib = None
_lock = threading.Lock()


def _bind(lib):
    p, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "sfft_version": ([], ctypes.c_int),
        "sfft_num_variants": ([i32, i32], ctypes.c_int),
        "sfft_build_twiddle_table": ([i32, i32, p, i64], ctypes.c_int),
        "sfft_plan_create": ([ctypes.POINTER(p), i32, i32, i32, i64, i32], ctypes.c_int),
        "sfft_plan_create_variant": ([ctypes.POINTER(p), i32, i32, i32, i64, i32, i32], ctypes.c_int),
        "sfft_plan_destroy": ([p], ctypes.c_int),
        "sfft_plan_info": ([p, ctypes.POINTER(PlanInfo)], ctypes.c_int),
        "sfft_plan_twiddles": ([p, p, i64], ctypes.c_int),
        "sfft_variant_info": ([i32, i32, i32, ctypes.POINTER(PlanInfo)], ctypes.c_int),
        "sfft_execute": ([p, p, p, i64, p, p], ctypes.c_int),
        "sfft_execute_sync": ([p, p, p, i64, p, ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
        "sfft_execute_ex": ([p, p, p, i64, p, p, i32], ctypes.c_int),
        "sfft_execute_sync_ex": ([p, p, p, i64, p, ctypes.POINTER(ctypes.c_float), i32], ctypes.c_int),
        "sfft_execute_host": ([p, p, p, i64], ctypes.c_int),
        "sfft_execute_host_ex": ([p, p, p, i64, i32], ctypes.c_int),
        "sfft_permute": ([i32, i32, p, p, p, i64, p], ctypes.c_int),
        "sfft_stage": ([i32, i32, i32, i32, i32, p, p, p, i64, p], ctypes.c_int),
        "sfft_last_error": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def lib():
    """The loaded library; raises FftError if it has not been built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    # a fresh checkout: compile the sm_100a library in-tree
                    # (nvcc is part of the image); never substitute a CPU path
                    try:
                        from .build import build

                        build()
                    except Exception as exc:  # noqa: BLE001
                        raise FftError(
                            f"native library {LIB_PATH} is missing and could not be built ({exc}); "
                            "build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                            "(there is no CPU fallback)"
                        ) from exc
                _lib = _bind(ctypes.CDLL(LIB_PATH))
    return _lib


def variant_info(n: int, precision_code: int, variant: int = 0) -> dict:
    """Kernel geometry of a variant, host-only (sfft_variant_info)."""
    info = PlanInfo()
    check(lib().sfft_variant_info(n, precision_code, variant, ctypes.byref(info)))
    return info.as_dict()


def check(status: int) -> None:
    """Raise the errors.py class matching a non-zero C-ABI status."""
    if status != 0:
        msg = lib().sfft_last_error().decode(errors="replace")
        raise STATUS_TO_ERROR.get(status, FftError)(msg)
