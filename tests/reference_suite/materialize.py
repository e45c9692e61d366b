"""Materialise the reference's own test suite (pkg/tests) for this package.

Test infrastructure only.  Copies ``/root/reference/pkg/tests/test_*.py``
into ``tests/reference_suite/vendored/`` as ``test_ref_<name>.py`` (renamed
so they cannot shadow this repo's own test modules of the same name) and
records the SHA-256 of every source in ``vendored/MANIFEST.json``.  The
directory is git-ignored -- the reference's files are not part of this
repository's history -- but not gpurun-ignored, so the suite travels to the
GPU box with the snapshot; ``__graft_entry__.build()`` refreshes it whenever
``/root/reference`` is present.  ``conftest.py`` next to this file maps
``stagefft`` onto ``paper_2203_09384_b200`` and lists the documented
deviations.

    python tests/reference_suite/materialize.py [--src /root/reference/pkg/tests]
"""

from __future__ import annotations

import argparse
import glob
import hashlib
import json
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "vendored")
DEFAULT_SRC = "/root/reference/pkg/tests"


def materialize(src: str = DEFAULT_SRC) -> list[str]:
    """Copy the suite; returns the written paths ([] if ``src`` is absent)."""
    sources = sorted(glob.glob(os.path.join(src, "test_*.py")))
    if not sources:
        return []
    os.makedirs(DEST, exist_ok=True)
    manifest, written = {}, []
    for path in sources:
        name = "test_ref_" + os.path.basename(path)[len("test_"):]
        target = os.path.join(DEST, name)
        shutil.copyfile(path, target)
        with open(path, "rb") as f:
            manifest[name] = {"source": path, "sha256": hashlib.sha256(f.read()).hexdigest()}
        written.append(target)
    with open(os.path.join(DEST, "MANIFEST.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    return written


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default=DEFAULT_SRC)
    for p in materialize(ap.parse_args().src):
        print(p)
