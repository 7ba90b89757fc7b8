"""Pin the CPU oracle (oracle/port.py, oracle/knnd_oracle.c) against the
golden vectors recorded from the reference itself (tests/golden/)."""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from oracle import native, port
from parity import sha_i32

SMALL = [
    "n300_d6_k7_s3", "n500_d5_k6_s23", "n2000_d6_k8_s20", "n1000_d20_k20_s1", "n1500_d16_k10_s7",
    "n600_d50_k30_s2", "n800_d10_k40_s5", "n5_d3_k4_s22", "n12_d3_k6_s4", "n4000_d5_k10_s0",
]
# the pure-Python port is slow (per-anchor loop); run it on the smaller cases
PORT_CASES = ["n300_d6_k7_s3", "n500_d5_k6_s23", "n600_d50_k30_s2", "n5_d3_k4_s22", "n12_d3_k6_s4",
              "n800_d10_k40_s5"]


def sha_f64(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# known answers (reference tests t_similarity:32-37, t_core:38-49, t_descent:44-62)


def test_kl_hand_values(known):
    pts = np.array(known["kl_points"])
    tab = port.KlTables(pts)
    assert tab.scores(0, np.array([1]))[0] == pytest.approx(0.5 * math.log(2.0) + 0.5 * math.log(2.0 / 3.0), rel=1e-12)
    assert tab.scores(0, np.array([1]))[0] == pytest.approx(known["kl_01"], rel=1e-15)
    assert tab.scores(0, np.array([2]))[0] == pytest.approx(known["kl_02"], rel=1e-15)
    assert tab.scores(1, np.array([0]))[0] == pytest.approx(known["kl_10"], rel=1e-15)
    assert known["kl_01"] == pytest.approx(0.143841, abs=1e-6)
    assert known["kl_02"] == pytest.approx(0.510826, abs=1e-6)


def test_batch_scores_pinned(known):
    pts = port.simplex_points(10, 300, np.random.default_rng(8))
    assert sha_f64(pts) == known["batch_points_sha"]
    tab = port.KlTables(pts)
    for x, ref in known["batch_scores"].items():
        assert np.array_equal(tab.scores(int(x)), np.array(ref))  # same einsum -> bitwise


def test_round_budget_pairs(known):
    for n, k, b in known["round_budget"]:
        assert port.budget(n, k) == b


def test_fcc_extremes(known):
    full = np.array([[1, 2], [0, 2], [0, 1]])
    assert port.fcc_rate(full, 500, 0, 1)[1] == known["fcc_complete"] == 1.0
    bip = np.array([[2, 3], [2, 3], [0, 1], [0, 1]])
    xs, i, j = port.fcc_draws(4, 2, 500, port.substream(1, 3, 1))
    assert port.fcc_count(bip, xs, i, j) == 0 == known["fcc_bipartite"]


# ---------------------------------------------------------------------------
# inputs: points and the initial digraph


@pytest.mark.parametrize("name", SMALL)
def test_points_and_init_match_reference(small_meta, small_tables, name):
    meta = small_meta[name]
    pts = port.experiment_points(meta["n"], meta["d"], meta["seed"])
    assert sha_f64(pts) == meta["points_sha"]
    draws = port.random_kout_draws(meta["n"], meta["k"], port.substream(meta["seed"], port.TAG_INIT))
    init_c = native.sort_rows(native.Tables(pts), draws)
    assert sha_i32(init_c) == meta["init_sha"]
    assert np.array_equal(init_c, small_tables[f"{name}/init"])


@pytest.mark.parametrize("name", PORT_CASES)
def test_port_init_matches_reference(small_meta, small_tables, name):
    meta = small_meta[name]
    pts = port.experiment_points(meta["n"], meta["d"], meta["seed"])
    draws = port.random_kout_draws(meta["n"], meta["k"], port.substream(meta["seed"], port.TAG_INIT))
    assert sha_i32(port.order_rows(port.KlTables(pts), draws)) == meta["init_sha"]


# ---------------------------------------------------------------------------
# whole trajectories


@pytest.mark.parametrize("name", SMALL)
def test_c_oracle_trajectory(small_meta, small_tables, name):
    meta = small_meta[name]
    pts = port.experiment_points(meta["n"], meta["d"], meta["seed"])
    shas = []
    final, hist = native.descend(native.Tables(pts), small_tables[f"{name}/init"], meta["seed"], 1000,
                                 port.round_cap(meta["n"], meta["k"]),
                                 on_round=lambda r, a, b: shas.append(sha_i32(b)))
    assert len(hist) == len(meta["rounds"])
    for h, r, s in zip(hist, meta["rounds"], shas):
        assert (h["comparisons"], h["changed"], h["fcc_count"]) == (r["comparisons"], r["changed"], r["fcc_count"])
        assert h["fcc"] == r["fcc"]
        assert s == r["sha"]
    assert np.array_equal(final, small_tables[f"{name}/final"])


@pytest.mark.parametrize("name", PORT_CASES)
def test_port_trajectory(small_meta, small_tables, name):
    meta = small_meta[name]
    pts = port.experiment_points(meta["n"], meta["d"], meta["seed"])
    final, hist = port.descend(pts, meta["k"], meta["seed"])
    assert [(h["comparisons"], h["changed"], h["fcc_count"]) for h in hist] == \
        [(r["comparisons"], r["changed"], r["fcc_count"]) for r in meta["rounds"]]
    assert sha_i32(final) == meta["rounds"][-1]["sha"]


def test_c_oracle_c1_trajectory(trajectories):
    ref = trajectories["c1"]
    pts = port.experiment_points(ref["n"], ref["d"], ref["seed"])
    tab = native.Tables(pts)
    draws = port.random_kout_draws(ref["n"], ref["k"], port.substream(ref["seed"], port.TAG_INIT))
    init = native.sort_rows(tab, draws)
    assert sha_i32(init) == ref["init_sha"]
    shas = []
    _, hist = native.descend(tab, init, ref["seed"], 1000, ref["max_rounds"],
                             on_round=lambda r, a, b: shas.append(sha_i32(b)))
    assert len(hist) == len(ref["rounds"])
    for h, r, s in zip(hist, ref["rounds"], shas):
        assert (h["comparisons"], h["changed"], h["fcc_count"], s) == \
            (r["comparisons"], r["changed"], r["fcc_count"], r["sha"])


def test_c_oracle_c2_round1(trajectories):
    """C2 (n=100k, d=10, K=20): init and round 1 bitwise equal to the reference."""
    ref = trajectories["c2"]
    pts = port.experiment_points(ref["n"], ref["d"], ref["seed"])
    assert sha_f64(pts) == ref["points_sha"]
    tab = native.Tables(pts)
    init = native.sort_rows(tab, port.random_kout_draws(ref["n"], ref["k"], port.substream(ref["seed"], 2)))
    assert sha_i32(init) == ref["init_sha"]
    rows, _, _, comps, changed = native.local_join(tab, init)
    r1 = ref["rounds"][0]
    assert (comps, changed, sha_i32(rows)) == (r1["comparisons"], r1["changed"], r1["sha"])


# ---------------------------------------------------------------------------
# transpose and exact neighbours


def test_transpose_matches_port():
    rng = np.random.default_rng(0)
    t = port.random_kout_draws(3000, 9, rng)
    ptr, idx = native.transpose(t)
    ptr2, idx2 = port.cofriend_csr(t)
    assert np.array_equal(ptr, ptr2) and np.array_equal(idx, idx2)


def test_exact_rows_match_port():
    pts = port.experiment_points(700, 6, 4)
    q = port.recall_sample(700, 0, 50)
    a = native.exact_rows(native.Tables(pts), q, 8)
    b = port.exact_rows(port.KlTables(pts), q, 8)
    assert np.array_equal(a, b)
