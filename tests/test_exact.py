"""GPU exact K-NN (knnd_exact_knn) against the C oracle's brute force
(oracle_exact_rows, pinned to evaluation.py:83-90 in test_oracle.py), and
recall at the BASELINE configs against the values recorded from the
reference's final tables (tests/golden/recall.json)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2202_00517_b200 as b2
from oracle import native, port

pytestmark = pytest.mark.gpu


def _check_rows(pts, queries, k):
    rs = b2.KlRankingSystem(pts, validate=False)
    got = b2.exact_rows(rs, queries, k)
    want = native.exact_rows(native.Tables(pts), np.asarray(queries), k)
    assert got.shape == want.shape
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert bad.size == 0, (bad[:5], got[bad[:2]], want[bad[:2]])
    return rs, got


@pytest.mark.parametrize("n,d,k,seed", [(10_000, 5, 10, 0), (3000, 20, 20, 1), (2000, 50, 30, 2),
                                         (1500, 10, 64, 3), (500, 16, 1, 4), (65, 8, 40, 5), (33, 3, 32, 6),
                                         (2, 3, 1, 7)])
def test_exact_rows_all_anchors(cuda, n, d, k, seed):
    pts = port.experiment_points(n, d, seed)
    _check_rows(pts, np.arange(n), k)


def test_exact_rows_sampled_c2(cuda):
    pts = port.experiment_points(100_000, 10, 0)
    q = port.recall_sample(100_000, 0, 10_000)[:2000]
    _check_rows(pts, q, 20)


def test_exact_scores_are_fp64_batch_scores(cuda):
    pts = port.experiment_points(3000, 20, 9)
    rs = b2.KlRankingSystem(pts, validate=False)
    q = np.array([0, 17, 2999])
    ids, sc = b2.evaluation.exact_rows_device(rs, q, 20, with_scores=True)
    ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
    for a, x in enumerate(q):
        full = rs.batch_scores(int(x))
        assert np.array_equal(sc[a], full[ids[a]])  # the same fp64 operator as batch_scores
        assert np.all(np.diff(sc[a]) >= 0)


def test_exact_rows_non_simplex(cuda):
    """coordinates > 1 (|x log y| accumulated separately, absolute error band)"""
    rng = np.random.default_rng(11)
    pts = rng.uniform(0.05, 3.0, size=(4000, 12))
    _check_rows(pts, rng.choice(4000, 500, replace=False), 15)


def test_exact_rows_duplicates_overflow_rerun(cuda):
    """400 copies of one point: every copy ties (score, id) with the others, so
    the candidate lists exceed the first capacity and are rerun"""
    pts = port.experiment_points(3000, 6, 12)
    pts[1000:1400] = pts[7]
    _check_rows(pts, np.array([7, 1000, 1399, 5, 2999]), 10)


def test_exact_knn_graph_and_recall_api(cuda):
    pts = port.experiment_points(2000, 8, 13)
    ds, rs = b2.Dataset(pts), b2.KlRankingSystem(pts)
    g = b2.exact_knn(ds, rs, 12)
    assert isinstance(g, b2.ExactKnnGraph) and g.n == 2000 and g.k == 12
    want = native.exact_rows(native.Tables(pts), np.arange(2000), 12)
    assert np.array_equal(g.neighbors, want)
    assert b2.recall(g.neighbors, g, np.arange(2000)) == 1.0
    friends, _ = b2.run(ds, rs, b2.DescentConfig(k=12, seed=0))
    sample = b2.uniform_recall_sample(2000, 0, 500)
    r = b2.recall(friends, g, sample)
    assert r == port.recall_of(friends, want[sample], sample)
    assert b2.sampled_recall(friends, rs, sample) == r
    with pytest.raises(b2.ConfigError):
        b2.exact_knn(b2.Dataset(pts[:5]), b2.KlRankingSystem(pts[:5]), 5)


@pytest.mark.parametrize("name,n,d,k", [("c2", 100_000, 10, 20), ("c3", 1_000_000, 20, 20),
                                        ("c4", 1_000_000, 50, 30)])
def test_recall_full_sample_matches_reference(cuda, trajectories, name, n, d, k):
    """recall of the reference's final table (rebuilt from the device descent,
    whose per-round tables match the reference's sha256) over the full
    10,000-id sample, with the exact rows from the GPU, equals the value
    recorded from the reference's own table and the C brute force."""
    from conftest import load_json

    rec = load_json("recall.json")
    if name not in rec:
        pytest.skip("no recorded recall")
    pts = port.experiment_points(n, d, 0)
    rs = b2.KlRankingSystem(pts, validate=False)
    friends, hist = b2.run(b2.Dataset(pts), rs, b2.DescentConfig(k=k, seed=0))
    assert len(hist) == len(trajectories[name]["rounds"])
    sample = port.recall_sample(n, 0, 10_000)
    assert b2.sampled_recall(friends, rs, sample) == rec[name]["recall"]
