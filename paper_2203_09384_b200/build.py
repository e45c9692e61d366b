"""In-tree build of the native library (sm_100a only).

``python -m paper_2203_09384_b200.build`` (or ``__graft_entry__.build()``)
compiles every ``csrc/*.cu`` translation unit to an object with nvcc -- in
parallel, one process per TU (the kernel instantiations are split by
precision and length across the ``sfft_table_*.cu`` units for this) -- and
links ``_lib/libsfft.so``.  The .so is git-ignored but travels to the GPU
box with the repo snapshot.
"""

from __future__ import annotations

import glob
import hashlib
import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libsfft.so")


def _sources() -> list:
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(CSRC, "*.cu")))


def _deps() -> list:
    return sorted(os.path.basename(p) for p in glob.glob(os.path.join(CSRC, "*")) if p.endswith((".cu", ".cuh", ".h")))

ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _fingerprint(flags) -> str:
    h = hashlib.sha256(" ".join(flags).encode())
    for name in _deps():
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(f.read())
    with open(os.path.join(ROOT, "include", "sfft.h"), "rb") as f:
        h.update(f.read())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(LIB_DIR, exist_ok=True)
    flags = [
        ARCH,
        "-O3",
        "-lineinfo",
        "-std=c++17",
        "-Xcompiler",
        "-fPIC",
        "-Xptxas",
        "-v" if verbose else "-O3",
    ]
    stamp_path = LIB_PATH + ".stamp"
    fp = _fingerprint(flags)
    if not force and os.path.exists(LIB_PATH) and os.path.exists(stamp_path):
        with open(stamp_path) as f:
            if f.read().strip() == fp:
                return LIB_PATH
    nvcc = _nvcc()
    with tempfile.TemporaryDirectory(prefix="sfft_build_") as tmpdir:

        def compile_one(src):
            obj = os.path.join(tmpdir, src.replace(".cu", ".o"))
            cmd = [nvcc, *flags, "-c", "-o", obj, os.path.join(CSRC, src)]
            proc = subprocess.run(cmd, capture_output=True, text=True)
            if proc.returncode != 0:
                raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
            if verbose:
                sys.stderr.write(proc.stderr)
            return obj

        with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as pool:
            objs = list(pool.map(compile_one, _sources()))
        tmp = LIB_PATH + ".tmp"
        cmd = [nvcc, ARCH, "-shared", "-o", tmp, *objs]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    os.replace(tmp, LIB_PATH)
    with open(stamp_path, "w") as f:
        f.write(fp)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
