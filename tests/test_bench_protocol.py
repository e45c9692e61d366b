"""Timing protocol (paper section 6.1) -- mirror of reference tests/test_bench.py.

Record/summary/export logic runs on CPU; run_benchmark drives the GPU and is
marked accordingly.
"""

import io
import json

import pytest

from paper_2203_09384_b200 import DomainError, InsufficientDataError
from paper_2203_09384_b200.bench import (
    RECORD_COLUMNS,
    BenchmarkRecord,
    export_records,
    export_summaries,
    flag_outliers,
    load_records,
    run_benchmark,
    summarize,
)


def record(length, iteration, total, warmup=False):
    return BenchmarkRecord(length=length, iteration=iteration, dispatch_us=total / 4,
                           compute_us=3 * total / 4, total_us=total, warmup=warmup)


def test_summary_basics_and_population_variance():
    (s,) = summarize([record(8, i, t) for i, t in enumerate([5.0, 3.0, 4.0])])
    assert s.mean_us == pytest.approx(4.0) and s.optimal_us == pytest.approx(3.0)
    assert s.iterations_kept == 3 and s.outliers_discarded == 0
    (s,) = summarize([record(8, i, t) for i, t in enumerate([2.0, 4.0])])
    assert s.variance_us2 == pytest.approx(1.0) and s.stddev_us == pytest.approx(1.0)


def test_outlier_rules():
    (s,) = summarize([record(8, i, t) for i, t in enumerate([10.0, 10.0, 10.0, 500.0])])
    assert s.outliers_discarded == 1 and s.mean_us == pytest.approx(10.0)
    assert s.optimal_us == pytest.approx(10.0)
    recs = [record(8, i, t) for i, t in enumerate([1.0, 1.0, 1.0, 1.0, 30.0])]
    assert summarize(recs, reference="median")[0].outliers_discarded == 1
    assert summarize(recs, reference="mean")[0].outliers_discarded == 0
    with pytest.raises(DomainError):
        flag_outliers(recs, outlier_factor=1.0)
    with pytest.raises(ValueError):
        flag_outliers(recs, reference="mode")


def test_warmups_never_flagged_and_all_warmup_raises():
    recs = [record(8, 0, 1000.0, warmup=True)] + [record(8, i, 1.0) for i in range(1, 4)]
    flagged = flag_outliers(recs)
    assert not flagged[0].outlier
    with pytest.raises(InsufficientDataError):
        summarize([record(8, 0, 1.0, warmup=True)])


def test_optimal_never_exceeds_mean_and_lengths_sorted():
    recs = [record(64, i, 1.0 + i) for i in range(5)] + [record(8, i, 2.0) for i in range(5)]
    sums = summarize(recs)
    assert [s.length for s in sums] == [8, 64]
    assert all(s.optimal_us <= s.mean_us for s in sums)


@pytest.mark.parametrize("fmt", ["csv", "json"])
def test_export_round_trip(tmp_path, fmt):
    recs = [record(8, 0, 0.1 + 0.2, warmup=True), record(8, 1, 1 / 3), record(16, 0, 1e-7)]
    recs = flag_outliers(recs)
    path = tmp_path / f"r.{fmt}"
    export_records(recs, path)
    assert load_records(path) == recs
    if fmt == "csv":
        assert path.read_text().splitlines()[0] == ",".join(RECORD_COLUMNS)


def test_export_header_only_and_summaries(tmp_path):
    buf = io.StringIO()
    export_records([], buf, format="csv")
    assert buf.getvalue().strip() == ",".join(RECORD_COLUMNS)
    path = tmp_path / "s.json"
    export_summaries(summarize([record(8, i, 2.0) for i in range(3)]), path, {"outlier_factor": 10.0})
    doc = json.loads(path.read_text())
    assert doc["metadata"]["variance"] == "population" and doc["summaries"][0]["length"] == 8
    with pytest.raises(ValueError):
        export_records([], tmp_path / "x.csv", format="xml")


def test_bad_iteration_counts():
    with pytest.raises(DomainError):
        run_benchmark([8], iterations=0)
    with pytest.raises(DomainError):
        run_benchmark([8], iterations=1, warmup_count=-1)


@pytest.mark.gpu
def test_run_benchmark_on_gpu(cuda):
    r = run_benchmark([8, 12, 4096, 1024], iterations=5, warmup_count=2)
    assert set(r.errors) == {12, 4096}
    assert {x.length for x in r.records} == {8, 1024}
    assert [x.warmup for x in r.records if x.length == 8] == [True, True] + [False] * 5
    assert all(x.compute_us > 0 and x.dispatch_us >= 0 for x in r.records)
    assert all(x.total_us == pytest.approx(x.dispatch_us + x.compute_us) for x in r.records)
    # deterministic GPU output -> checksums stable across runs (test_bench.py:41-46)
    r2 = run_benchmark([8, 1024], iterations=2, warmup_count=0)
    assert r2.checksums == {k: v for k, v in r.checksums.items()}
    # device-resident, batched, double precision
    r3 = run_benchmark([2048], iterations=3, warmup_count=1, precision="double", batch=64,
                       signal="random", device=cuda)
    assert len(r3.records) == 4 and len(summarize(r3.records)) == 1
