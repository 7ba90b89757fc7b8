"""The reference's acceptance criteria C1-C7 (tests/test_acceptance.py of the
reference package; the statistical ones over five seeds, four to pass) run
through this package's harness mirror and device engine.  C6, which the
reference itself fails (18/50), is checked as parity with the reference's
per-instance results instead.  C8/C9 exercise the metrizability checker, which
is out of scope here."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2202_00517_b200 as b2
from paper_2202_00517_b200 import bench as xb

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SEEDS = (0, 1, 2, 3, 4)


@pytest.fixture(scope="module")
def k16_runs(cuda):
    return [xb.run_experiment(xb.ExperimentSpec(n=20_000, d=10, k=16, seed=s, recall_mode="full")) for s in SEEDS]


@pytest.fixture(scope="module")
def k32_runs(cuda):
    return [xb.run_experiment(xb.ExperimentSpec(n=20_000, d=10, k=32, seed=s, recall_mode="off")) for s in SEEDS]


@pytest.fixture(scope="module")
def sweep_runs(cuda):
    return xb.dimension_sweep(xb.ExperimentSpec(n=20_000, d=10, k=16, seed=7, recall_mode="full"), [10, 20, 40, 60])


@pytest.fixture(scope="module")
def scaling_runs(cuda):
    return {n: xb.run_experiment(xb.ExperimentSpec(n=n, d=10, k=16, seed=11, recall_mode="off"))
            for n in (10_000, 40_000)}


def test_c1_oracle_recall(k16_runs):
    assert sum(r.recall >= 0.90 for r in k16_runs) >= 4, [r.recall for r in k16_runs]


def test_c2_round_bound(k16_runs, k32_runs):
    assert sum(r.rounds_used <= 8 for r in k16_runs) >= 4
    assert sum(r.rounds_used <= 6 for r in k32_runs) >= 4


def test_c3_fcc_trajectory(k16_runs):
    ok = 0
    for rep in k16_runs:
        rates = [r.fcc for r in rep.rounds]
        rising = all(b > a for a, b in zip(rates[:-2], rates[1:-1]))
        ok += rates[0] < 0.05 and rising and 0.22 <= rates[-1] <= 0.32
    assert ok >= 4


def test_c4_dimension_decline(sweep_runs):
    by_d = {r.spec.d: r for r in sweep_runs}
    assert by_d[10].recall > by_d[20].recall > by_d[60].recall
    fccs = [by_d[d].final_fcc for d in (10, 20, 40, 60)]
    assert all(a >= b for a, b in zip(fccs, fccs[1:])), fccs


def test_c5_determinism_under_workers(cuda):
    maps = [xb.run_experiment(xb.ExperimentSpec(n=5_000, d=10, k=8, seed=5, recall_mode="off", workers=w)).friend_map
            for w in (1, 4, "auto")]
    assert np.array_equal(maps[0], maps[1]) and np.array_equal(maps[0], maps[2])


def test_c6_small_instance_equivalence_matches_reference(cuda):
    """The 50 Gaussian instances (n ~ U[20, 200], K in {2, 4, 8}, d in 2..5) run
    to a fixed point.  The reference's own criterion (recall 1.0 in >= 45) fails
    in the reference too: its recorded run (test_output.txt) and a rerun here
    give 18/50, every run at a true fixed point.  Parity is what is checked: per
    instance the same final table, round count and recall as the reference
    (tests/golden/c6_cases.json, make_c6_golden.py)."""
    import hashlib

    from conftest import load_json

    golden = load_json("c6_cases.json")
    gen = np.random.default_rng(606)
    exact, non_fixed = 0, 0
    for i in range(50):
        n = int(gen.integers(20, 201))
        k = int(gen.choice([2, 4, 8]))
        d = int(gen.integers(2, 6))
        pts = gen.standard_normal((n, d))
        ds, rs = b2.Dataset(pts), b2.EuclideanRankingSystem(pts)
        friends, hist = b2.run_to_fixed_point(ds, rs, b2.DescentConfig(k=k, seed=i, max_rounds=1000))
        rec = b2.recall(friends, b2.exact_knn(ds, rs, k), np.arange(n))
        g = golden[i]
        assert (g["n"], g["k"], g["d"]) == (n, k, d)
        assert hashlib.sha256(np.ascontiguousarray(friends, dtype=np.int32).tobytes()).hexdigest() == g["sha"], i
        assert len(hist) == g["rounds"] and rec == g["recall"], i
        exact += rec == 1.0
        non_fixed += hist[-1].changed_friend_sets != 0
    assert exact == sum(c["recall"] == 1.0 for c in golden) == 18 and non_fixed == 0


def test_c7_complexity_instrumentation(k16_runs, k32_runs, sweep_runs, scaling_runs):
    worst = max(max(r.comparisons for r in rep.rounds) / (3 * rep.spec.n * (rep.spec.k + 2 * rep.spec.k ** 2))
                for rep in list(k16_runs) + list(k32_runs) + list(sweep_runs) + list(scaling_runs.values()))
    assert worst <= 1.0
    ratio = scaling_runs[40_000].rounds[0].comparisons / scaling_runs[10_000].rounds[0].comparisons
    assert 3.0 <= ratio <= 5.0
