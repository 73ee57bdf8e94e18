"""Harness-compatible benchmark rows for the GPU path.

Mirrors the reference harness's report format and protocol
(/root/reference/pkg/src/roaringset/bench/harness.py): rows with the columns
``dataset, structure, benchmark, metric, value, units, runs, dispersion``
(harness.py:34-35,43-71), a correctness-gated warm-up that aborts timing on
any disagreement (harness.py:230-235), then the median of >= 5 timed runs
(harness.py:114-123) reported as ns per input value over the successive
pairs of a dataset (bench_pairwise, harness.py:205-239).  GPU runs are timed
with CUDA events on the library stream, so GPU and CPU rows share one report.
"""

from __future__ import annotations

import csv
import json
import statistics
import sys
from dataclasses import asdict, dataclass

import numpy as np

from . import _lib
from .batch import BitmapBatch
from .containers import OPS

CSV_COLUMNS = ("dataset", "structure", "benchmark", "metric", "value", "units", "runs", "dispersion")
DISPERSION_FLAG = 1.10


class CorrectnessError(RuntimeError):
    """The GPU result disagreed with the expected cardinalities; timing aborted."""


@dataclass
class BenchRow:
    dataset: str
    structure: str
    benchmark: str
    metric: str
    value: float
    units: str
    runs: int
    dispersion: float


class BenchReport:
    def __init__(self, rows=None):
        self.rows: list[BenchRow] = list(rows or [])

    def extend(self, rows) -> None:
        self.rows.extend(rows)

    def to_csv(self, fh) -> None:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        for r in self.rows:
            w.writerow([r.dataset, r.structure, r.benchmark, r.metric, f"{r.value:.6g}", r.units, r.runs,
                        f"{r.dispersion:.4g}"])

    def to_json(self, fh) -> None:
        json.dump([asdict(r) for r in self.rows], fh, indent=2)
        fh.write("\n")


def _measure_gpu(work, runs: int):
    """Median of >= 5 device-timed runs (ns) and max/min dispersion."""
    reps = max(int(runs), 5)
    times = []
    for _ in range(reps):
        _lib.synchronize()
        e0 = _lib.Event()
        work()
        e1 = _lib.Event()
        times.append(e0.elapsed_ms(e1) * 1e6)
    med = float(statistics.median(times))
    return med, max(times) / max(min(times), 1e-9), reps


def bench_pairwise(name: str, batch: BitmapBatch, op: str, expected_cards, count_only: bool = False,
                   runs: int = 5, structure: str = "roaring-b200") -> list[BenchRow]:
    """bench_pairwise over successive pairs (i, i+1) of `batch`, reported in ns
    per input value.  `expected_cards` are the oracle cardinalities of the
    pairs (harness.py:214); a mismatch raises CorrectnessError before timing."""
    if op not in OPS:
        raise ValueError(f"unknown op {op!r}")
    n = len(batch)
    if n < 2:
        raise CorrectnessError("pairwise benchmark needs at least two sets")
    ia, ib = np.arange(n - 1), np.arange(1, n)
    cards = batch.cardinalities().astype(np.int64)
    denom = int(cards[:-1].sum() + cards[1:].sum())

    def work():
        if count_only:
            return batch.pairwise_cardinality(op, batch, ia, ib)
        return batch.pairwise(op, batch, ia, ib)

    got = work()
    got = got if count_only else got.cardinalities()
    got = np.asarray(got, dtype=np.int64)
    expected = np.asarray(expected_cards, dtype=np.int64)
    if not np.array_equal(got, expected):
        bad = int(np.flatnonzero(got != expected)[0])
        raise CorrectnessError(f"{structure} {op}: pair {bad} cardinality {got[bad]} != oracle {expected[bad]}")
    med, disp, reps = _measure_gpu(work, runs)
    metric = f"{op}_count" if count_only else op
    if disp > DISPERSION_FLAG:
        print(f"warning: {name}/{structure}/{metric} dispersion {disp:.3f} exceeds {DISPERSION_FLAG}",
              file=sys.stderr)
    return [BenchRow(name, structure, "pairwise", metric, med / max(denom, 1), "ns/value", reps, disp)]


def bench_wide_union(name: str, batch: BitmapBatch, expected_card: int, runs: int = 5,
                     structure: str = "roaring-b200") -> list[BenchRow]:
    """bench_wide_union (harness.py:243-266): union_many over all bitmaps."""
    denom = int(batch.cardinalities().sum())
    got = int(batch.union_many().cardinalities()[0])
    if got != int(expected_card):
        raise CorrectnessError(f"{structure} wide union cardinality {got} != oracle {expected_card}")
    med, disp, reps = _measure_gpu(lambda: batch.union_many(), runs)
    return [BenchRow(name, structure, "wideunion", "wideunion", med / max(denom, 1), "ns/value", reps, disp)]
