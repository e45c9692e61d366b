"""C-ABI boundary checks that need no GPU.

* the shared library loads and exports every function include/sfft.h declares;
* the header is plain C (a C program compiled with gcc links and runs against
  it, so no C++ or torch type leaks through the boundary);
* argument validation returns the status codes of the reference exception
  tree before any device is touched.
"""

import ctypes
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

from paper_2203_09384_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sfft.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfft_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    if shutil.which("nm"):
        out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
        exported = set(re.findall(r"\bT (sfft_\w+)", out))
        assert set(declared_functions()) <= exported


def test_plain_c_client(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("gcc missing")
    src = tmp_path / "client.c"
    src.write_text(
        """
#include <stdio.h>
#include "sfft.h"
int main(void) {
  float tw[16];
  sfft_plan_t plan = 0;
  int v = sfft_version();
  int rc = sfft_build_twiddle_table(8, SFFT_SINGLE, tw, sizeof(tw));
  int bad = sfft_plan_create(&plan, 12, SFFT_SINGLE, SFFT_FORWARD, 0, 0);
  printf("%d %d %d %.7f %.7f %s\\n", v, rc, bad, tw[2], tw[3], sfft_last_error());
  return rc;
}
"""
    )
    exe = tmp_path / "client"
    subprocess.run(
        ["gcc", "-std=c99", "-Wall", "-Werror", str(src), "-I", os.path.join(ROOT, "include"),
         "-L", _native.LIB_DIR, "-lsfft", f"-Wl,-rpath,{_native.LIB_DIR}", "-o", str(exe)],
        check=True,
    )
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out[0] == "100" and out[1] == "0" and out[2] == "1"
    assert abs(float(out[3]) - np.sqrt(0.5)) < 1e-7 and abs(float(out[4]) + np.sqrt(0.5)) < 1e-7


def test_status_codes_before_device():
    lib = _native.lib()
    h = ctypes.c_void_p()
    assert lib.sfft_plan_create(ctypes.byref(h), 12, 0, 0, 0, 0) == 1  # InvalidLengthError
    assert lib.sfft_plan_create(ctypes.byref(h), 4096, 0, 0, 0, 0) == 2  # UnsupportedLengthError
    assert lib.sfft_plan_create(ctypes.byref(h), 1, 0, 0, 0, 0) == 2
    assert lib.sfft_plan_create(ctypes.byref(h), 64, 5, 0, 0, 0) == 7  # bad precision
    assert lib.sfft_plan_create(ctypes.byref(h), 64, 0, 9, 0, 0) == 7  # bad direction
    assert lib.sfft_plan_create(ctypes.byref(h), 64, 0, 0, -1, 0) == 4  # ShapeError
    assert lib.sfft_plan_create_variant(ctypes.byref(h), 64, 0, 0, 0, 0, 42) == 3  # PlanError
    assert lib.sfft_plan_create(None, 64, 0, 0, 0, 0) == 7
    assert b"power of two" in lib.sfft_last_error() or lib.sfft_last_error()
    assert lib.sfft_execute(None, None, None, 1, None, None) == 7
    assert lib.sfft_execute_host(None, None, None, 1) == 7
    assert lib.sfft_plan_destroy(None) == 0
    assert lib.sfft_num_variants(12, 0) == 0 and lib.sfft_num_variants(64, 0) >= 1


def test_check_maps_status_to_reference_errors():
    import paper_2203_09384_b200 as sf

    lib = _native.lib()
    h = ctypes.c_void_p()
    with pytest.raises(sf.UnsupportedLengthError):
        _native.check(lib.sfft_plan_create(ctypes.byref(h), 4096, 0, 0, 0, 0))
    with pytest.raises(sf.InvalidLengthError):
        _native.check(lib.sfft_plan_create(ctypes.byref(h), 12, 0, 0, 0, 0))


def test_last_error_is_thread_local():
    import threading

    lib = _native.lib()
    h = ctypes.c_void_p()
    lib.sfft_plan_create(ctypes.byref(h), 12, 0, 0, 0, 0)
    mine = lib.sfft_last_error()
    seen = []

    def other():
        seen.append(lib.sfft_last_error())

    t = threading.Thread(target=other)
    t.start()
    t.join()
    assert seen == [b""] and mine


def test_no_gpu_means_loud_cuda_error():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2203_09384_b200 as sf

    with pytest.raises(sf.CudaError):
        sf.execute(sf.make_plan(64), np.ones(64, np.complex64))
