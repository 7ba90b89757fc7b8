"""Squared-Euclidean scorer (EuclideanRankingSystem, similarity.py:119-140)
through the same fused join: the C oracle pinned to the reference's own
Euclidean trajectories (tests/golden/l2_trajectories.json, make_l2_golden.py),
then the GPU against both (``-m gpu``)."""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, load_json
from oracle import native, port

sys.path.insert(0, GOLDEN)
from make_l2_golden import CASES, vectors  # noqa: E402


def sha(t) -> str:
    return hashlib.sha256(np.ascontiguousarray(t, dtype="<i4").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def l2_golden():
    return load_json("l2_trajectories.json")


def _oracle_trajectory(name):
    n, d, k, seed, kind = CASES[name]
    tab = native.L2Tables(vectors(n, d, seed, kind))
    draws = port.random_kout_draws(n, k, port.substream(seed, port.TAG_INIT))
    init = native.sort_rows(tab, draws)
    final, hist = native.descend(tab, init, seed, 1000, port.round_cap(n, k))
    return tab, init, final, hist


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_l2_matches_reference_trajectory(l2_golden, name):
    g = l2_golden[name]
    n, d, k, seed, kind = CASES[name]
    tab, init, final, hist = _oracle_trajectory(name)
    assert sha(init) == g["init_sha"]
    assert len(hist) == len(g["rounds"])
    for h, r in zip(hist, g["rounds"]):
        assert (h["comparisons"], h["changed"], h["fcc_count"]) == (r["comparisons"], r["changed"], r["fcc_count"])
    assert sha(native.exact_rows(tab, np.arange(n), k)) == g["exact_sha"]


# ---------------------------------------------------------------------------
# GPU


@pytest.fixture(params=["q23", "fp32"])
def screen(request, monkeypatch):
    """Both screens of the join: the 23-bit fixed-point rows (default where they exist) and the fp32 rows."""
    monkeypatch.setenv("KNND_Q23", "1" if request.param == "q23" else "0")
    return request.param


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_l2_trajectory_matches_reference(cuda, l2_golden, name, screen):
    import paper_2202_00517_b200 as b2

    g = l2_golden[name]
    n, d, k, seed, kind = CASES[name]
    v = vectors(n, d, seed, kind)
    rs = b2.EuclideanRankingSystem(v)
    cfg = b2.DescentConfig(k=k, seed=seed)
    st = b2.init_random_kout(b2.Dataset(v), rs, cfg, b2.derive_rng(seed, 2))
    assert sha(st.friends) == g["init_sha"]
    for r in g["rounds"]:
        st, s = b2.run_round(st, rs, cfg)
        assert s.round_index == r["round"]
        assert (s.comparisons, s.changed_friend_sets) == (r["comparisons"], r["changed"]), r["round"]
        assert round(s.fcc * cfg.fcc_sample_count) == r["fcc_count"]
        assert sha(st.friends) == r["sha"], r["round"]
    friends, hist = b2.run(b2.Dataset(v), rs, cfg)
    assert len(hist) == len(g["rounds"]) and sha(friends) == g["rounds"][-1]["sha"]
    ex = b2.exact_knn(b2.Dataset(v), rs, k)
    assert sha(ex.neighbors) == g["exact_sha"]
    assert b2.recall(friends, ex, np.arange(n)) == g["recall"]


@pytest.mark.gpu
def test_gpu_l2_batch_scores_and_join_vs_oracle(cuda, screen):
    import paper_2202_00517_b200 as b2

    v = vectors(4000, 12, 21, "normal") * 3.0 + 5.0
    rs = b2.EuclideanRankingSystem(v)
    assert (rs.device_tables().q23 is not None) == (screen == "q23")
    tab = native.L2Tables(v)
    full = rs.batch_scores(17)
    d2 = np.maximum(tab.xlogx[17] + tab.xlogx - 2.0 * (v @ v[17]), 0.0)
    np.testing.assert_allclose(full, d2, rtol=1e-12, atol=1e-9)
    ids = np.array([3, 17, 3999])
    assert np.array_equal(rs.batch_scores(17, ids), full[ids])
    # one round from a random table: rows, |U| and tallies equal the C oracle's
    k = 16
    draws = port.random_kout_draws(4000, k, port.substream(5, port.TAG_INIT))
    init = native.sort_rows(tab, draws)
    st = b2.KnnState(init)
    nxt, s = b2.run_round(st, rs, b2.DescentConfig(k=k, seed=5))
    rows, _, _, comps, changed = native.local_join(tab, init)
    assert np.array_equal(nxt.friends, rows)
    assert (s.comparisons, s.changed_friend_sets) == (comps, changed)
    q = np.arange(0, 4000, 7)
    assert np.array_equal(b2.exact_rows(rs, q, k), native.exact_rows(tab, q, k))


@pytest.mark.gpu
def test_gpu_l2_accepts_reference_style_system(cuda):
    """device_tables_for takes any object named EuclideanRankingSystem exposing
    .vectors (and ._sq), as a reference instance does."""
    import paper_2202_00517_b200 as b2

    class EuclideanRankingSystem:  # stand-in with the reference's attributes
        def __init__(self, vecs):
            self.vectors = vecs
            self._sq = np.einsum("ij,ij->i", vecs, vecs)

    v = vectors(1500, 6, 22, "uniform")
    a, _ = b2.run(b2.Dataset(v), EuclideanRankingSystem(v), b2.DescentConfig(k=8, seed=1))
    b, _ = b2.run(b2.Dataset(v), b2.EuclideanRankingSystem(v), b2.DescentConfig(k=8, seed=1))
    assert np.array_equal(a, b)


@pytest.mark.gpu
def test_gpu_l2_extreme_scales_keep_fp32_rows(cuda):
    """The Q23 weights 2 (x - mu) h 2^126 must stay in fp32's normal range: data of an
    extreme scale screen the fp32 rows, and the tables still equal the oracle's."""
    import paper_2202_00517_b200 as b2

    base = vectors(1500, 10, 3, "normal")
    for scale, q23 in ((1.0, True), (1e6, False), (1e-40, False)):
        v = base * scale
        rs = b2.EuclideanRankingSystem(v)
        assert (rs.device_tables().q23 is not None) == q23, scale
        k = 10
        tab = native.L2Tables(v)
        init = native.sort_rows(tab, port.random_kout_draws(1500, k, port.substream(2, port.TAG_INIT)))
        nxt, s = b2.run_round(b2.KnnState(init), rs, b2.DescentConfig(k=k, seed=2))
        rows, _, _, comps, changed = native.local_join(tab, init)
        assert np.array_equal(nxt.friends, rows), scale
        assert (s.comparisons, s.changed_friend_sets) == (comps, changed)
