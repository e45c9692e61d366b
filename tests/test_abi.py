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


C_GPU_CLIENT = r"""
#include <complex.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include "sfft.h"
/* plain-C caller: plan, host execute, compare with a direct DFT in double */
int main(void) {
  const int n = 256, batch = 33;
  float* x = malloc(sizeof(float) * 2 * n * batch);
  float* y = malloc(sizeof(float) * 2 * n * batch);
  for (int i = 0; i < 2 * n * batch; ++i) x[i] = (float)((i * 7919 % 1000) / 500.0 - 1.0);
  sfft_plan_t plan;
  int rc = sfft_plan_create(&plan, n, SFFT_SINGLE, SFFT_FORWARD, batch, 0);
  if (rc) { printf("create %d %s\n", rc, sfft_last_error()); return 1; }
  rc = sfft_execute_host(plan, x, y, batch);
  if (rc) { printf("execute %d %s\n", rc, sfft_last_error()); return 1; }
  double worst = 0;
  for (int b = 0; b < batch; b += 8) {
    double num = 0, den = 0;
    for (int k = 0; k < n; ++k) {
      double complex acc = 0;
      for (int m = 0; m < n; ++m) {
        double a = -2.0 * M_PI * (double)((long)k * m % n) / n;
        acc += (x[2 * (b * n + m)] + I * x[2 * (b * n + m) + 1]) * cexp(I * a);
      }
      double complex got = y[2 * (b * n + k)] + I * y[2 * (b * n + k) + 1];
      num += pow(cabs(got - acc), 2); den += pow(cabs(acc), 2);
    }
    if (sqrt(num / den) > worst) worst = sqrt(num / den);
  }
  x[5] = NAN;
  int dom = sfft_execute_host(plan, x, y, batch);
  sfft_plan_destroy(plan);
  printf("%.3e %d\n", worst, dom);
  return worst < 8e-5 && dom == SFFT_ERR_DOMAIN ? 0 : 2;
}
"""


@pytest.mark.gpu
def test_plain_c_client_on_gpu(tmp_path, cuda):
    src = tmp_path / "gpu_client.c"
    src.write_text(C_GPU_CLIENT)
    exe = tmp_path / "gpu_client"
    subprocess.run(
        ["gcc", "-std=gnu99", "-O2", str(src), "-I", os.path.join(ROOT, "include"), "-L", _native.LIB_DIR,
         "-lsfft", f"-Wl,-rpath,{_native.LIB_DIR}", "-lm", "-o", str(exe)],
        check=True,
    )
    res = subprocess.run([str(exe)], capture_output=True, text=True)
    assert res.returncode == 0, res.stdout + res.stderr
