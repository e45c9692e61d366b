"""The paper's timing protocol (section 6.1) as the reference's ``bench`` module.

Reference contract (bench.py:26-307): one plan and one input per length;
``warmup_count + iterations`` timed executions recorded in order; the
leading warm-ups are flagged, never dropped; a non-warm-up record is an
outlier when its total exceeds ``outlier_factor`` x the median (or mean) of
its length's non-warm-up totals; summaries average the kept records with
the population variance, while the optimum is the minimum over every
non-warm-up record, outliers included; the SHA-256 of each length's
(deterministic) output is recorded once; CSV/JSON export round-trips
exactly.

Here the records come from the GPU path: ``dispatch_us`` is the host time
up to the kernel launch (validation, dtype conversion and, for host input,
the H2D copy), ``compute_us`` the device time from CUDA events (plus the D2H
copy for host input).  ``run_benchmark`` adds ``precision``, ``batch`` and
``device`` so the same protocol covers the paper's single-transform latency
table and batched throughput runs.

The record table is column-driven: ``_COLUMNS`` gives each exported column
its text encoder and decoder, and both formats are generated from it.
"""

from __future__ import annotations

import csv
import hashlib
import io
import json
import math
import os
from dataclasses import asdict, dataclass, replace
from typing import Callable, NamedTuple

import numpy as np

from .errors import DomainError, InsufficientDataError, InvalidLengthError, PlanError
from .executor import execute_timed
from .planner import Algorithm, Direction, make_plan
from .signalgen import generate, generate_batch


@dataclass(frozen=True)
class BenchmarkRecord:
    """One timed execution."""

    length: int
    iteration: int
    dispatch_us: float
    compute_us: float
    total_us: float
    warmup: bool
    outlier: bool = False


@dataclass(frozen=True)
class BenchmarkSummary:
    """Statistics of one length over its kept (non-warm-up, non-outlier) records."""

    length: int
    iterations_kept: int
    mean_us: float
    variance_us2: float  # population variance (divide by the kept count)
    stddev_us: float
    optimal_us: float    # min total over ALL non-warm-up records
    outliers_discarded: int


class BenchmarkResult(NamedTuple):
    """Records in execution order, per-length planning errors, per-length output SHA-256."""

    records: list
    errors: dict
    checksums: dict


# ------------------------------------------------------------------ columns
class _Column(NamedTuple):
    name: str
    to_text: Callable[[object], str]
    from_text: Callable[[str], object]
    from_json: Callable[[object], object]


def _bool_text(v) -> str:
    return "true" if v else "false"


_COLUMNS = (
    _Column("length", str, int, int),
    _Column("iteration", str, int, int),
    _Column("warmup", _bool_text, lambda s: s == "true", bool),
    _Column("outlier", _bool_text, lambda s: s == "true", bool),
    _Column("dispatch_us", repr, float, float),  # repr: shortest exact round trip
    _Column("compute_us", repr, float, float),
    _Column("total_us", repr, float, float),
)

#: exported column order (also the CSV header)
RECORD_COLUMNS = tuple(c.name for c in _COLUMNS)
EXPORT_FORMATS = ("csv", "json")


def _format_of(path, explicit: str | None) -> str:
    fmt = explicit or ("json" if os.path.splitext(str(path))[1].lower() == ".json" else "csv")
    if fmt not in EXPORT_FORMATS:
        raise ValueError(f"unknown export format {fmt!r}; expected one of {EXPORT_FORMATS}")
    return fmt


# ---------------------------------------------------------------- protocol
def _bench_input(signal: str, length: int, seed: int, precision: str, batch, device):
    if batch is None:
        x = generate(signal, length, seed, precision)
    elif signal == "random":
        x = generate_batch(batch, length, seed, precision)
    else:
        x = np.broadcast_to(generate(signal, length, seed, precision), (batch, length)).copy()
    if device is None:
        return x
    import torch

    return torch.from_numpy(x).to(device)


def _sha256(output) -> str:
    host = output.detach().cpu().numpy() if hasattr(output, "detach") else np.asarray(output)
    return hashlib.sha256(np.ascontiguousarray(host).tobytes()).hexdigest()


def run_benchmark(
    lengths,
    iterations: int = 1000,
    warmup_count: int = 1,
    algorithm: Algorithm = Algorithm.MIXED_RADIX,
    signal: str = "ramp",
    seed: int = 0,
    *,
    precision: str = "single",
    batch: int | None = None,
    device=None,
) -> BenchmarkResult:
    """Time ``warmup_count + iterations`` forward transforms per length (bench.py:85-129).

    ``device=None`` feeds numpy input (host -> GPU -> host per call, the
    reference's calling convention); a device such as ``"cuda:0"`` keeps the
    input resident.  Lengths that cannot be planned are reported in
    ``errors`` and the others still run.
    """
    if iterations < 1:
        raise DomainError(f"iterations must be >= 1, got {iterations}")
    if warmup_count < 0:
        raise DomainError(f"warmup_count must be >= 0, got {warmup_count}")
    result = BenchmarkResult([], {}, {})
    for n in map(int, lengths):
        try:
            plan = make_plan(n, Direction.FORWARD, algorithm, precision=precision)
        except (InvalidLengthError, PlanError) as exc:
            result.errors[n] = str(exc)
            continue
        x = _bench_input(signal, n, seed, precision, batch, device)
        for it in range(warmup_count + iterations):
            out, dispatch, compute = execute_timed(plan, x)
            if n not in result.checksums:
                result.checksums[n] = _sha256(out)
            result.records.append(
                BenchmarkRecord(n, it, dispatch, compute, dispatch + compute, warmup=it < warmup_count)
            )
    return result


def _center(values: list, reference: str) -> float:
    if reference == "median":
        return float(np.median(np.asarray(values, dtype=np.float64)))
    return math.fsum(values) / len(values)


def flag_outliers(records, outlier_factor: float = 10.0, reference: str = "median") -> list:
    """The records with ``outlier`` recomputed, order preserved, inputs untouched (bench.py:132-160)."""
    if not outlier_factor > 1.0:
        raise DomainError(f"outlier_factor must be > 1, got {outlier_factor}")
    if reference not in ("median", "mean"):
        raise ValueError(f"reference must be 'median' or 'mean', got {reference!r}")
    timed: dict[int, list] = {}
    for r in records:
        if not r.warmup:
            timed.setdefault(r.length, []).append(r.total_us)
    limit = {n: outlier_factor * _center(v, reference) for n, v in timed.items()}
    out = []
    for r in records:
        want = bool(not r.warmup and r.total_us > limit[r.length])
        out.append(r if r.outlier == want else replace(r, outlier=want))
    return out


def summarize(records, outlier_factor: float = 10.0, reference: str = "median") -> list:
    """One :class:`BenchmarkSummary` per length, ascending (bench.py:163-199)."""
    by_length: dict[int, list] = {}
    for r in flag_outliers(records, outlier_factor, reference):
        if not r.warmup:
            by_length.setdefault(r.length, []).append(r)
        else:
            by_length.setdefault(r.length, [])
    summaries = []
    for n in sorted(by_length):
        measured = by_length[n]
        if not measured:
            raise InsufficientDataError(f"length {n}: every record is a warm-up; nothing to summarize")
        kept = [r.total_us for r in measured if not r.outlier]
        mean = math.fsum(kept) / len(kept)
        var = math.fsum((t - mean) ** 2 for t in kept) / len(kept)
        summaries.append(
            BenchmarkSummary(
                length=n,
                iterations_kept=len(kept),
                mean_us=mean,
                variance_us2=var,
                stddev_us=math.sqrt(var),
                optimal_us=min(r.total_us for r in measured),
                outliers_discarded=len(measured) - len(kept),
            )
        )
    return summaries


# ------------------------------------------------------------------- export
def _records_text(records, fmt: str) -> str:
    rows = [asdict(r) for r in records]
    if fmt == "json":
        return json.dumps([{c.name: row[c.name] for c in _COLUMNS} for row in rows], indent=2) + "\n"
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(RECORD_COLUMNS)
    w.writerows([c.to_text(row[c.name]) for c in _COLUMNS] for row in rows)
    return buf.getvalue()


def _write_text(destination, text: str, newline=None) -> None:
    if hasattr(destination, "write"):
        destination.write(text)
        return
    with open(destination, "w", encoding="utf-8", newline=newline) as fp:
        fp.write(text)


def export_records(records, destination, format: str | None = None) -> None:
    """Per-iteration records as CSV (``RECORD_COLUMNS`` header, repr floats,
    true/false booleans; zero records = header only) or a JSON list, to a
    path or an open text file (bench.py:207-245)."""
    fmt = _format_of(destination, format)
    _write_text(destination, _records_text(records, fmt), newline="")


def _record_from(values: dict, decode: str) -> BenchmarkRecord:
    return BenchmarkRecord(**{c.name: getattr(c, decode)(values[c.name]) for c in _COLUMNS})


def load_records(source, format: str | None = None) -> list:
    """Read what :func:`export_records` wrote (bench.py:248-287)."""
    fmt = _format_of(source, format)
    with open(source, encoding="utf-8", newline="") as fp:
        text = fp.read()
    if fmt == "json":
        return [_record_from(row, "from_json") for row in json.loads(text)]
    reader = csv.reader(text.splitlines())
    header = next(reader, None)
    if header is None or tuple(header) != RECORD_COLUMNS:
        raise DomainError(f"unexpected record CSV header: {header!r}")
    return [_record_from(dict(zip(RECORD_COLUMNS, row)), "from_text") for row in reader if row]


def export_summaries(summaries, destination, metadata: dict | None = None) -> None:
    """``{"metadata": {...}, "summaries": [...]}`` as JSON (bench.py:290-307).

    ``metadata`` always records the variance convention ("population")."""
    doc = {"metadata": dict({"variance": "population"}, **(metadata or {})),
           "summaries": [asdict(s) for s in summaries]}
    _write_text(destination, json.dumps(doc, indent=2) + "\n")
