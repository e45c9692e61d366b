import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def rel_l2(a, b) -> float:
    """tests/test_executor.py:18-19 of the reference."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def row_rel_l2(a, b) -> np.ndarray:
    a = np.asarray(a).astype(np.complex128)
    b = np.asarray(b).astype(np.complex128)
    return np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)


def tolerance(n: int, precision: str) -> float:
    """north_star: rel-L2 <= 1e-5*log2(N) fp32, <= 1e-13*log2(N) fp64."""
    return (1e-5 if precision == "single" else 1e-13) * np.log2(n)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))

    return load


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
