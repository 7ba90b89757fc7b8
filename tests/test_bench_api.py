"""The experiment harness mirror (paper_2202_00517_b200.bench) against the
reference's own reports (tests/golden/bench_reports.json, recorded by
make_bench_golden.py from rankdescent.bench, bench.py:136-267)."""

import numpy as np
import pytest

from conftest import load_json

import paper_2202_00517_b200 as b2
from paper_2202_00517_b200 import ConfigError, RoundStats
from paper_2202_00517_b200 import bench as xb


@pytest.fixture(scope="module")
def golden():
    return load_json("bench_reports.json")


def fixed_report(rec):
    """Our report object rebuilt from a golden record with the golden's fixed clock."""
    spec = xb.ExperimentSpec(**rec["spec"])
    rounds = [RoundStats(r, 0.25 * (i + 1), f, c, ch) for i, (r, f, c, ch) in enumerate(rec["rounds"])]
    return xb.ExperimentReport(spec=spec, rounds=rounds, rounds_used=rec["rounds_used"],
                               round_budget=rec["round_budget"], final_fcc=rec["final_fcc"], recall=rec["recall"],
                               total_duration_sec=1.5)


def test_emit_report_matches_reference_bytes(golden):
    for rec in golden["reports"]:
        rep = fixed_report(rec)
        assert xb.emit_report(rep, "json") == rec["emit_json"]
        assert xb.emit_report(rep, "csv") == rec["emit_csv"]
        assert xb.emit_report(rep) == rec["emit_" + rep.spec.output_format]


def test_emit_sweep_matches_reference_bytes(golden):
    sw = golden["sweep"]
    reps = [fixed_report(r) for r in sw["reports"]]
    assert xb.emit_sweep(reps, "json") == sw["emit_json"]
    assert xb.emit_sweep(reps, "csv") == sw["emit_csv"]
    with pytest.raises(ConfigError, match="unknown format"):
        xb.emit_sweep(reps, "xml")
    with pytest.raises(ConfigError, match="unknown format"):
        xb.emit_report(reps[0], "xml")


@pytest.mark.parametrize("kw, msg", [
    (dict(n=10, d=3, k=1), "need n > k >= 2"),
    (dict(n=5, d=3, k=5), "need n > k >= 2"),
    (dict(n=50, d=1, k=3), "need d >= 2"),
    (dict(n=50, d=3, k=3, ranking="cosine"), "ranking must be one of"),
    (dict(n=50, d=3, k=3, recall_mode="half"), "recall_mode must be one of"),
    (dict(n=50, d=3, k=3, output_format="xml"), "output_format must be one of"),
])
def test_spec_validation(kw, msg):
    with pytest.raises(ConfigError, match=msg):
        xb.ExperimentSpec(**kw)


def test_oracle_guard_before_any_work():
    with pytest.raises(xb.OracleGuardError, match="exceeds the guard of 100000"):
        xb.run_experiment(xb.ExperimentSpec(n=100_001, d=3, k=4))
    with pytest.raises(ConfigError, match="does not match spec"):
        import numpy as np

        xb.run_experiment(xb.ExperimentSpec(n=50, d=3, k=4, recall_mode="off"), points=np.ones((50, 4)) / 4)


def test_descent_config_mapping():
    s = xb.ExperimentSpec(n=100, d=3, k=7, seed=5, fcc_samples=33, max_rounds=2, workers="auto")
    c = s.descent_config()
    assert (c.k, c.fcc_sample_count, c.max_rounds, c.seed, c.worker_count) == (7, 33, 2, 5, "auto")


@pytest.mark.gpu
def test_run_experiment_matches_reference(golden, cuda):
    for rec in golden["reports"]:
        rep = xb.run_experiment(xb.ExperimentSpec(**rec["spec"]))
        got = [[r.round_index, r.fcc, r.comparisons, r.changed_friend_sets] for r in rep.rounds]
        assert got == rec["rounds"], rec["spec"]
        assert (rep.rounds_used, rep.round_budget, rep.final_fcc, rep.recall) == (
            rec["rounds_used"], rec["round_budget"], rec["final_fcc"], rec["recall"]), rec["spec"]
        assert rep.friend_map.shape == (rec["spec"]["n"], rec["spec"]["k"])
        assert rep.total_duration_sec > 0


@pytest.mark.gpu
def test_dimension_sweep_matches_reference(golden, cuda):
    sw = golden["sweep"]
    reps = xb.dimension_sweep(xb.ExperimentSpec(**sw["base"]), sw["dims"])
    assert [r.spec.d for r in reps] == sw["dims"]
    for rep, rec in zip(reps, sw["reports"]):
        got = [[r.round_index, r.fcc, r.comparisons, r.changed_friend_sets] for r in rep.rounds]
        assert got == rec["rounds"]
        assert (rep.rounds_used, rep.final_fcc, rep.recall) == (rec["rounds_used"], rec["final_fcc"], rec["recall"])


def _small(**kw):
    base = dict(n=300, d=5, k=6, seed=3)
    base.update(kw)
    return xb.ExperimentSpec(**base)


@pytest.mark.gpu
def test_report_shape_and_reproducibility(cuda):
    """bench.py behaviours the reference's test_bench.py pins: report fields,
    reproducible modulo wall clock, worker count and singleton sweeps change
    nothing, recall modes, parseable CSV rows."""
    import csv
    import io
    import json

    a = xb.run_experiment(_small())
    assert a.rounds_used == len(a.rounds) >= 1 and a.round_budget == b2.round_budget(300, 6)
    assert a.final_fcc == a.rounds[-1].fcc and 0.0 <= a.recall <= 1.0 and a.friend_map.shape == (300, 6)
    b = xb.run_experiment(_small(workers=4))
    assert np.array_equal(a.friend_map, b.friend_map) and a.recall == b.recall
    assert [r.comparisons for r in a.rounds] == [r.comparisons for r in b.rounds]
    (swept,) = xb.dimension_sweep(_small(), [5])
    assert np.array_equal(swept.friend_map, a.friend_map) and swept.recall == a.recall
    assert xb.run_experiment(_small(recall_mode="off")).recall is None
    assert xb.run_experiment(_small(ranking="euclidean")).recall > 0.5
    obj = json.loads(xb.emit_report(a, "json"))
    assert obj["summary"]["final_fcc"] == a.final_fcc and obj["summary"]["recall"] == a.recall
    rows = list(csv.DictReader(io.StringIO(xb.emit_report(a, "csv"))))
    assert len(rows) == a.rounds_used + 1 and rows[-1]["record"] == "summary"
    assert [int(r["round_index"]) for r in rows[:-1]] == list(range(1, a.rounds_used + 1))
