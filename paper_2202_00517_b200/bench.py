"""Experiment runner on the B200 engine — mirrors the reference's bench.py
(generate data, run descent, measure, report; bench.py:1-267).

``run_experiment(ExperimentSpec(...))`` keeps the reference's spec fields,
validation messages, timed region (init + rounds, bench.py:155-157), report
fields and JSON / CSV serialisation byte for byte, so a caller of
``rankdescent.bench`` can switch imports.  What differs is underneath: the
descent is ``paper_2202_00517_b200.run`` (device rounds) and the recall ground
truth is the GPU brute force (``evaluation.exact_rows``).  For the default
``sample6`` mode only the sampled anchors' exact rows are computed — the same
recall value the reference gets from its full O(n^2) oracle (bench.py:160-166)
— and ``full`` computes every row on the GPU.  The oracle guard
(``OracleGuardError`` above 100,000 points without ``force_oracle``,
bench.py:141-145) is kept for drop-in behaviour, even though the GPU oracle
makes it cheap.
"""

from __future__ import annotations

import csv
import dataclasses
import io
import json
import logging
import time
from dataclasses import dataclass, field

import numpy as np

from .core import ConfigError, Dataset
from .descent import STREAM_DATA, DescentConfig, RoundStats, derive_rng, round_budget, run
from .evaluation import ExactKnnGraph, exact_knn, exact_rows, recall, uniform_recall_sample
from .similarity import EuclideanRankingSystem, KlRankingSystem, sample_simplex_uniform

logger = logging.getLogger(__name__)

ORACLE_GUARD = 100_000  # evaluation.py:32
RANKINGS = ("kl", "euclidean")
RECALL_MODES = ("sample6", "full", "off")
FORMATS = ("json", "csv")


class OracleGuardError(RuntimeError):
    """bench.py:40-41 — recall would run the quadratic oracle above the guard."""


@dataclass
class ExperimentSpec:
    """bench.py:45-83 — parameters of one run; (spec, seed) reproduces everything."""

    n: int
    d: int
    k: int
    seed: int = 0
    ranking: str = "kl"
    fcc_samples: int = 1000
    max_rounds: int | None = None
    workers: int | str = 1
    recall_mode: str = "sample6"
    output_format: str = "json"
    force_oracle: bool = False

    def __post_init__(self) -> None:
        if self.k < 2 or self.n <= self.k:
            raise ConfigError(f"need n > k >= 2, got n={self.n}, k={self.k}")
        if self.d < 2:
            raise ConfigError(f"need d >= 2, got d={self.d}")
        if self.ranking not in RANKINGS:
            raise ConfigError(f"ranking must be one of {RANKINGS}, got {self.ranking!r}")
        if self.recall_mode not in RECALL_MODES:
            raise ConfigError(f"recall_mode must be one of {RECALL_MODES}, got {self.recall_mode!r}")
        if self.output_format not in FORMATS:
            raise ConfigError(f"output_format must be one of {FORMATS}, got {self.output_format!r}")

    def descent_config(self) -> DescentConfig:
        return DescentConfig(k=self.k, fcc_sample_count=self.fcc_samples, max_rounds=self.max_rounds,
                             seed=self.seed, worker_count=self.workers)

    def to_dict(self) -> dict:
        return dataclasses.asdict(self)


@dataclass
class ExperimentReport:
    """bench.py:86-125 — per-round stats plus the scaling-table summary."""

    spec: ExperimentSpec
    rounds: list[RoundStats]
    rounds_used: int
    round_budget: int
    final_fcc: float
    recall: float | None
    total_duration_sec: float
    friend_map: np.ndarray | None = field(repr=False, compare=False, default=None)  # in-memory only

    @property
    def first_round_sec(self) -> float:
        return self.rounds[0].wall_clock_sec

    @property
    def last_round_sec(self) -> float:
        return self.rounds[-1].wall_clock_sec

    def summary_dict(self) -> dict:
        return {
            "rounds_used": self.rounds_used,
            "round_budget": self.round_budget,
            "final_fcc": self.final_fcc,
            "recall": self.recall,
            "total_duration_sec": self.total_duration_sec,
            "first_round_sec": self.first_round_sec,
            "last_round_sec": self.last_round_sec,
        }

    def to_json_obj(self) -> dict:
        return {"spec": self.spec.to_dict(), "rounds": [dataclasses.asdict(r) for r in self.rounds],
                "summary": self.summary_dict()}


def generate_points(spec: ExperimentSpec) -> np.ndarray:
    """bench.py:125-127 — uniform simplex points from the (seed, data, d) substream."""
    return sample_simplex_uniform(spec.d, spec.n, derive_rng(spec.seed, STREAM_DATA, spec.d))


def make_ranking_system(spec: ExperimentSpec, points: np.ndarray):
    """bench.py:130-133."""
    if spec.ranking == "kl":
        return KlRankingSystem(points, validate=False)
    return EuclideanRankingSystem(points)


def _recall(spec: ExperimentSpec, dataset: Dataset, rs, friends: np.ndarray) -> float:
    """bench.py:160-166 on the GPU oracle: only the rows the recall reads."""
    if spec.recall_mode == "full":
        return recall(friends, exact_knn(dataset, rs, spec.k), np.arange(spec.n))
    sample = uniform_recall_sample(spec.n, spec.seed)
    rows = np.zeros((spec.n, spec.k), dtype=np.int64)
    rows[sample] = exact_rows(rs, sample, spec.k)
    return recall(friends, ExactKnnGraph(rows), sample)


def run_experiment(spec: ExperimentSpec, points: np.ndarray | None = None) -> ExperimentReport:
    """bench.py:136-185.  Timed region: initialization and rounds only; data
    generation and the exact oracle are excluded."""
    if spec.recall_mode != "off" and spec.n > ORACLE_GUARD and not spec.force_oracle:
        raise OracleGuardError(
            f"exact oracle on n={spec.n} exceeds the guard of {ORACLE_GUARD}; "
            "set force_oracle (or recall_mode='off') to proceed"
        )
    if points is None:
        points = generate_points(spec)
    if points.shape != (spec.n, spec.d):
        raise ConfigError(f"points shape {points.shape} does not match spec ({spec.n}, {spec.d})")
    dataset = Dataset(points)
    rs = make_ranking_system(spec, points)

    t0 = time.perf_counter()
    friends, rounds = run(dataset, rs, spec.descent_config())
    total = time.perf_counter() - t0

    recall_value = None if spec.recall_mode == "off" else _recall(spec, dataset, rs, friends)
    report = ExperimentReport(spec=spec, rounds=rounds, rounds_used=len(rounds),
                              round_budget=round_budget(spec.n, spec.k), final_fcc=rounds[-1].fcc,
                              recall=recall_value, total_duration_sec=total, friend_map=friends)
    logger.info(
        "experiment n=%d d=%d k=%d ranking=%s seed=%d: rounds=%d/%d fcc=%.4f recall=%s time=%.2fs",
        spec.n, spec.d, spec.k, spec.ranking, spec.seed, report.rounds_used, report.round_budget,
        report.final_fcc, "n/a" if recall_value is None else f"{recall_value:.4f}", total,
    )
    return report


def dimension_sweep(base: ExperimentSpec, dims: list[int]) -> list[ExperimentReport]:
    """bench.py:187-192 — one report per dimension, descent seed held fixed."""
    if not dims:
        raise ConfigError("dims must be nonempty")
    return [run_experiment(dataclasses.replace(base, d=d)) for d in dims]


# ---------------------------------------------------------------------------
# serialisation (bench.py:197-267): same columns, same cell formatting

_CSV_HEADER = [
    "record", "round_index", "wall_clock_sec", "fcc", "comparisons", "changed_friend_sets",
    "n", "d", "k", "seed", "ranking", "fcc_samples", "max_rounds", "workers", "recall_mode",
    "rounds_used", "round_budget", "final_fcc", "recall",
    "total_duration_sec", "first_round_sec", "last_round_sec",
]

_SWEEP_HEADER = [
    "d", "n", "k", "seed", "ranking", "rounds_used", "round_budget",
    "final_fcc", "recall", "total_duration_sec", "first_round_sec", "last_round_sec",
]


def _cell(value) -> str:
    if value is None:
        return ""
    if isinstance(value, float):
        return format(value, ".17g")  # round-trips through float()
    return str(value)


def _csv(rows: list[list]) -> str:
    buf = io.StringIO()
    csv.writer(buf, lineterminator="\n").writerows(rows)
    return buf.getvalue()


def emit_report(report: ExperimentReport, fmt: str | None = None) -> str:
    """bench.py:218-244 — JSON object, or CSV round rows plus a summary row."""
    fmt = fmt or report.spec.output_format
    if fmt == "json":
        return json.dumps(report.to_json_obj(), indent=2)
    if fmt != "csv":
        raise ConfigError(f"unknown format {fmt!r}")
    spec, s = report.spec, report.summary_dict()
    pad = [""] * (len(_CSV_HEADER) - 6)
    rows = [_CSV_HEADER]
    rows += [[_cell(v) for v in ("round", r.round_index, r.wall_clock_sec, r.fcc, r.comparisons,
                                 r.changed_friend_sets)] + pad for r in report.rounds]
    rows.append(["summary", "", "", "", "", ""] + [_cell(v) for v in (
        spec.n, spec.d, spec.k, spec.seed, spec.ranking, spec.fcc_samples, spec.max_rounds, spec.workers,
        spec.recall_mode, s["rounds_used"], s["round_budget"], s["final_fcc"], s["recall"],
        s["total_duration_sec"], s["first_round_sec"], s["last_round_sec"])])
    return _csv(rows)


def emit_sweep(reports: list[ExperimentReport], fmt: str) -> str:
    """bench.py:247-267 — JSON report list, or one CSV row per dimension."""
    if fmt == "json":
        return json.dumps({"dims": [r.spec.d for r in reports], "reports": [r.to_json_obj() for r in reports]},
                          indent=2)
    if fmt != "csv":
        raise ConfigError(f"unknown format {fmt!r}")
    rows = [_SWEEP_HEADER]
    rows += [[_cell(v) for v in (r.spec.d, r.spec.n, r.spec.k, r.spec.seed, r.spec.ranking, r.rounds_used,
                                 r.round_budget, r.final_fcc, r.recall, r.total_duration_sec, r.first_round_sec,
                                 r.last_round_sec)] for r in reports]
    return _csv(rows)
