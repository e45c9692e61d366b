"""Stage-level API on the GPU vs the reference stage functions (oracle port).

Mirrors reference tests/test_kernels.py: single butterflies, radix-4 ramp,
radix-8 impulse/constant, N = 8/16 pipelines with every stage order, inverse
round trip, argument validation; plus fp64 pipelines and batches.
"""

import numpy as np
import pytest

import oracle
import paper_2203_09384_b200 as sf
from conftest import rel_l2, row_rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def run_pipeline(x, stages, direction="forward", precision="single"):
    """Digit-reverse, fold the radix stages left to right (tests/test_kernels.py:25-36)."""
    x = np.asarray(x)
    n = x.shape[-1]
    table = sf.build_twiddle_table(n, precision)
    buf = sf.StageBuffer(sf.digit_reverse(x, stages, precision), 1)
    for i, r in enumerate(stages):
        buf = sf.kernels.RADIX_STAGE[r](buf, table, i, direction)
    out = buf.data
    return out / n if direction == "inverse" else out


def test_single_butterflies_and_small_kats(cuda):
    t2 = sf.build_twiddle_table(2)
    out = sf.radix2_stage(sf.StageBuffer(np.array([1, 1], np.complex64), 1), t2, 0)
    np.testing.assert_allclose(out.data, [2, 0], atol=1e-7)
    assert out.stride == 2
    np.testing.assert_allclose(sf.radix2_stage(sf.StageBuffer(np.array([1, 2], np.complex64), 1), t2, 0).data,
                               [3, -1], atol=1e-7)
    t4 = sf.build_twiddle_table(4)
    np.testing.assert_allclose(sf.radix4_stage(sf.StageBuffer(np.arange(4, dtype=np.complex64), 1), t4, 0).data,
                               [6, -2 + 2j, -2, -2 - 2j], atol=1e-6)
    t8 = sf.build_twiddle_table(8)
    imp = np.zeros(8, np.complex64)
    imp[0] = 1
    np.testing.assert_allclose(sf.radix8_stage(sf.StageBuffer(imp, 1), t8, 0).data, np.ones(8), atol=1e-6)
    np.testing.assert_allclose(sf.radix8_stage(sf.StageBuffer(np.ones(8, np.complex64), 1), t8, 0).data,
                               8 * imp, atol=1e-6)


@pytest.mark.parametrize("stages", [[2, 2, 2], [8], [8, 2], [2, 8], [4, 4], [2, 2, 2, 2], [8, 8, 8, 4], [4, 2, 8]])
@pytest.mark.parametrize("precision", ["single", "double"])
def test_pipelines_match_oracle_stage_engine(cuda, stages, precision):
    n = int(np.prod(stages))
    dt = np.complex64 if precision == "single" else np.complex128
    x = oracle.generate_batch(17, n, seed=n, dtype=dt)
    for d in ("forward", "inverse"):
        got = run_pipeline(x, stages, d, precision)
        want = oracle.mixed_radix_execute(x, d, stages=stages, dtype=dt)
        tol = (1e-5 if precision == "single" else 1e-13) * np.log2(n)
        assert row_rel_l2(got, want).max() <= tol
        assert row_rel_l2(got, oracle.direct_dft(x, d)).max() <= tol


def test_stage_on_device_tensors_and_out(cuda):
    x = torch.from_numpy(oracle.generate_batch(4, 64, 1)).cuda()
    t = sf.build_twiddle_table(64)
    out = torch.empty_like(x)
    buf = sf.radix8_stage(sf.StageBuffer(sf.digit_reverse(x, [8, 8]), 1), t, 0, out=out)
    assert buf.data is out and buf.data.is_cuda and buf.stride == 8
    y = sf.radix8_stage(buf, t, 1).data
    assert rel_l2(y.cpu().numpy(), oracle.direct_dft(x.cpu().numpy())) <= 1e-5


def test_stage_validation(cuda):
    t8 = sf.build_twiddle_table(8)
    with pytest.raises(sf.PlanError):
        sf.radix8_stage(sf.StageBuffer(np.ones(8, np.complex64), 2), t8, 0)
    with pytest.raises(sf.PlanError):
        sf.radix2_stage(sf.StageBuffer(np.ones(8, np.complex64), 3), t8, 0)
    with pytest.raises(sf.PlanError):
        sf.radix2_stage(sf.StageBuffer(np.ones(8, np.complex64), 1), sf.build_twiddle_table(16), 0)
    with pytest.raises(sf.PlanError):
        sf.radix2_stage(sf.StageBuffer(np.ones(8, np.complex64), 1), t8, 0, out=np.empty(4, np.complex64))
    data = np.arange(8, dtype=np.complex64)
    snap = data.copy()
    sf.radix4_stage(sf.StageBuffer(data, 1), t8, 0)
    assert np.array_equal(data, snap)
