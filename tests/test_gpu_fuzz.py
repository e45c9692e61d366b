"""Randomised GPU parity (hypothesis): any length, batch, precision, direction
and compiled kernel variant, with signal magnitudes spanning many decades,
against the oracle port of the reference and the exact complex128 DFT.

Complements tests/test_gpu_parity.py (fixed grid of cases) with shapes nobody
picked by hand: batches that leave every kind of partial CTA / warp tile /
persistent-grid tail, offsets into a larger buffer, and rows scaled by 2^-60
.. 2^60 (the relative tolerance must hold at every scale).
"""

import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import paper_2203_09384_b200 as sf
from conftest import row_rel_l2, tolerance

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@st.composite
def cases(draw):
    p = draw(st.integers(1, 11))
    prec = draw(st.sampled_from(["single", "double"]))
    nvar = sf._native.lib().sfft_num_variants(2**p, 0 if prec == "single" else 1)
    return {
        "n": 2**p,
        "prec": prec,
        "direction": draw(st.sampled_from(["forward", "inverse"])),
        "variant": draw(st.integers(0, nvar - 1)),
        "batch": draw(st.integers(1, max(1, 40000 // 2**p))),
        "offset": draw(st.integers(0, 3)),  # rows skipped in front: misaligned-to-CTA bases
        "log_scale": draw(st.integers(-60, 60)),
        "seed": draw(st.integers(0, 2**31 - 1)),
    }


@settings(max_examples=int(os.environ.get("SFFT_FUZZ_EXAMPLES", "120")), deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(cases())
def test_random_shapes_match_oracle(cuda, c):
    n, prec = c["n"], c["prec"]
    dtype = np.complex64 if prec == "single" else np.complex128
    rows = c["batch"] + c["offset"]
    x = sf.generate_batch(rows, n, seed=c["seed"], precision=prec)
    x = (x * np.float64(2.0) ** c["log_scale"]).astype(dtype)
    plan = sf.make_plan(n, c["direction"], precision=prec, variant=c["variant"])
    xd = torch.from_numpy(x).to(cuda)
    got = sf.execute(plan, xd[c["offset"]:]).cpu().numpy()
    sub = x[c["offset"]:]
    want = oracle.reference_execute(sub, c["direction"], dtype=dtype)
    exact = oracle.direct_dft(sub, c["direction"])
    tol = tolerance(n, prec)
    assert row_rel_l2(got, exact).max() <= tol
    assert row_rel_l2(got, want).max() <= tol


@settings(max_examples=int(os.environ.get("SFFT_FUZZ_EXAMPLES_HOST", "60")), deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(p=st.integers(1, 11), prec=st.sampled_from(["single", "double"]),
       direction=st.sampled_from(["forward", "inverse"]), batch=st.integers(0, 3000),
       pinned=st.booleans(), seed=st.integers(0, 2**31 - 1))
def test_host_path_equals_device_path(cuda, p, prec, direction, batch, pinned, seed):
    """numpy in -> numpy out (sfft_execute_host: small-call bounce path or the
    chunked pipeline, pageable or pinned) is bit-identical to the device path,
    for 1-D (batch 0 means a single (N,) signal) and 2-D inputs."""
    n = 2**p
    x = sf.generate_batch(max(batch, 1), n, seed=seed, precision=prec)
    if batch == 0:
        x = x[0]
    if pinned:
        x = torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
    plan = sf.make_plan(n, direction, precision=prec)
    host = sf.execute(plan, x)
    dev = sf.execute(plan, torch.from_numpy(np.ascontiguousarray(x)).to(cuda)).cpu().numpy()
    assert host.shape == x.shape and host.dtype == x.dtype
    assert np.array_equal(host, dev)
