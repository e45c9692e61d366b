"""Regenerate the golden fixtures from the reference package itself.

Run in the development container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

Every output here comes from calling the reference ``stagefft`` functions
directly -- ``execute``/``make_plan`` (executor.py:50-96, planner.py:139-188),
``split_radix_transform`` (kernels.py:205-232), the radix stage functions on
complex128 buffers (the fp64 recipe of SURVEY.md 8(c)), ``generate``
(signalgen.py:14-41), ``digit_reversal_permutation`` (planner.py:62-89),
``build_twiddle_table`` (numerics.py:55-71) and ``FourierTransformer``
(estimator.py:19-78).  The committed ``.npz`` files travel to the GPU box;
this script does not.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = os.environ.get("STAGEFFT_SRC", "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

KINDS = ("random", "ramp", "impulse", "constant")
ENGINE_LENGTHS = tuple(2**p for p in range(3, 12))
ALL_LENGTHS = tuple(2**p for p in range(1, 12))
STAGE_LISTS = ([2, 2, 2], [4, 4], [8, 2], [2, 8], [8, 8, 8, 4], [4, 2, 8], [2] * 11, [8, 8, 8, 2])


def _fp64_restatement(sf, x, direction):
    """SURVEY.md 8(c) fp64 recipe, built only from reference functions."""
    n = x.shape[0]
    a = (-2 * np.pi / n) * np.arange(n, dtype=np.float64)
    f = np.cos(a) + 1j * np.sin(a)
    f[0] = 1
    table = sf.TwiddleTable(n, f)
    stages = sf.factorize_stages(n) if n >= 8 else [2] * (n.bit_length() - 1)
    stage_fn = {2: sf.radix2_stage, 4: sf.radix4_stage, 8: sf.radix8_stage}
    buf = sf.StageBuffer(x[sf.digit_reversal_permutation(stages)].astype(np.complex128), 1)
    for i, r in enumerate(stages):
        buf = stage_fn[r](buf, table, i, direction)
    out = buf.data
    if direction is sf.Direction.INVERSE:
        out = out / n
    return out


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import stagefft as sf  # the reference package, imported read-only

    # 1. engine outputs (complex64), N = 8..2048, four kinds, both directions
    eng = {}
    for n in ENGINE_LENGTHS:
        for kind in KINDS:
            x = sf.generate(kind, n, seed=n)
            eng[f"in_{kind}_{n}"] = x
            for d in ("forward", "inverse"):
                eng[f"out_{kind}_{n}_{d}"] = sf.execute(sf.make_plan(n, d), x)
    # split-radix route: the reference's only engine path for N = 2, 4
    for n in (2, 4, 8, 16, 64):
        x = sf.generate("random", n, seed=100 + n)
        eng[f"in_split_{n}"] = x
        for d in ("forward", "inverse"):
            eng[f"out_split_{n}_{d}"] = sf.split_radix_transform(
                x, sf.build_twiddle_table(n), sf.Direction(d)
            )
    np.savez_compressed(os.path.join(HERE, "engine_c64.npz"), **eng)

    # 2. fp64 restatement outputs, N = 2..2048, both directions
    f64 = {}
    for n in ALL_LENGTHS:
        rng = np.random.Generator(np.random.Philox(key=7 * n))
        parts = rng.uniform(-1.0, 1.0, size=(2, n))
        x = parts[0] + 1j * parts[1]
        f64[f"in_{n}"] = x
        for d in ("forward", "inverse"):
            f64[f"out_{n}_{d}"] = _fp64_restatement(sf, x, sf.Direction(d))
    np.savez_compressed(os.path.join(HERE, "restated_c128.npz"), **f64)

    # 3. plan-time constants: factorisations, permutations, twiddle tables
    plan = {}
    for n in ENGINE_LENGTHS:
        plan[f"stages_{n}"] = np.array(sf.factorize_stages(n))
    for stages in STAGE_LISTS:
        key = "_".join(map(str, stages))
        plan[f"perm_{key}"] = np.asarray(sf.digit_reversal_permutation(stages))
    for p in range(0, 13):
        plan[f"twiddle_{2**p}"] = sf.build_twiddle_table(2**p).factors
    np.savez_compressed(os.path.join(HERE, "plan_constants.npz"), **plan)

    # 4. batched caller: FourierTransformer (row loop over execute)
    rng = np.random.default_rng(0)
    X = (rng.uniform(-1, 1, (5, 64)) + 1j * rng.uniform(-1, 1, (5, 64))).astype(np.complex64)
    est = sf.FourierTransformer().fit(X)
    Y = est.transform(X)
    np.savez_compressed(
        os.path.join(HERE, "estimator_c64.npz"), X=X, Y=Y, Xback=est.inverse_transform(Y)
    )

    # 5. inputs: reference generate("random") for a few (n, seed) pairs
    gen = {f"random_{n}_{s}": sf.generate("random", n, seed=s) for n in (8, 1024) for s in (0, 1, 42)}
    np.savez_compressed(os.path.join(HERE, "signals_c64.npz"), **gen)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
