"""Property-based checks of the host logic (hypothesis; CPU only)."""

import math

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
import paper_2203_09384_b200 as sf

radix_lists = st.lists(st.sampled_from([2, 4, 8]), min_size=1, max_size=5)


@settings(max_examples=60, deadline=None)
@given(radix_lists)
def test_digit_reversal_bijection_and_oracle_agreement(stages):
    perm = sf.digit_reversal_permutation(stages)
    n = math.prod(stages)
    assert sorted(perm.tolist()) == list(range(n))
    assert np.array_equal(perm, oracle.digit_reversal_permutation(stages))


@settings(max_examples=200, deadline=None)
@given(st.integers(0, 10**7), st.integers(1, 64))
def test_shard_bounds_cover_exactly(batch, world):
    spans = [sf.shard_bounds(batch, world, r) for r in range(world)]
    covered = sum(b - a for a, b in spans)
    assert covered == batch
    assert all(a <= b for a, b in spans)
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


@settings(max_examples=40, deadline=None)
@given(st.integers(1, 11), st.sampled_from(["forward", "inverse"]), st.sampled_from(["mixed", "split"]),
       st.sampled_from(["single", "double"]))
def test_make_plan_fields(p, direction, algorithm, precision):
    n = 2**p
    plan = sf.make_plan(n, direction, algorithm, precision=precision)
    assert plan == sf.make_plan(n, sf.Direction(direction), sf.Algorithm(algorithm), precision=sf.Precision(precision))
    assert math.prod(plan.stages) == n and plan.chunk == n
    assert plan.scale == (1.0 / n if direction == "inverse" else 1.0)
    assert sf.count_butterflies(plan) == (n // 2) * p
    info = sf._native.variant_info(n, plan.precision.code, 0)
    assert math.prod(info["radices"]) == n


@settings(max_examples=30, deadline=None)
@given(st.integers(1, 4096), st.integers(0, 2**31 - 1))
def test_generate_batch_row0_is_generate(n, seed):
    assert np.array_equal(sf.generate_batch(1, n, seed)[0], sf.generate("random", n, seed))
    assert np.array_equal(sf.generate_batch(1, n, seed)[0], oracle.generate("random", n, seed))
