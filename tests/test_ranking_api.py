"""The ranking systems and the exact K-NN / recall API on the device,
restating the reference's own test_similarity.py / test_evaluation.py checks
(batch_scores orders and batch independence, Euclidean ties, exact_knn on
line points / the forced case / a dense divergence matrix, recall) against
independent host oracles (scipy rel_entr, numpy distances)."""

from __future__ import annotations

import numpy as np
import pytest
from scipy.special import rel_entr

import paper_2202_00517_b200 as b2

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------------------
# KlRankingSystem (similarity.py:80-116)


def test_kl_identity_and_hand_values(cuda):
    rs = b2.KlRankingSystem(np.array([[0.5, 0.5], [0.25, 0.75], [0.5, 0.5]]))
    assert rs.score(0, 2) == pytest.approx(0.0, abs=1e-15)
    assert rs.score(0, 1) == pytest.approx(0.143841, abs=1e-6)
    assert rs.score(1, 0) == pytest.approx(0.130812, abs=1e-6)


def test_kl_matches_scipy_rel_entr(cuda):
    pts = b2.sample_simplex_uniform(8, 60, 1)
    rs = b2.KlRankingSystem(pts)
    for x in (0, 17, 59):
        ref = np.array([rel_entr(pts[x], pts[y]).sum() for y in range(60)])
        np.testing.assert_allclose(rs.batch_scores(x), ref, rtol=1e-12, atol=1e-15)


def test_kl_order_matches_divergence_matrix_argsort(cuda):
    pts = b2.sample_simplex_uniform(6, 40, 5)
    rs = b2.KlRankingSystem(pts)
    dmat = np.array([[rel_entr(pts[i], pts[j]).sum() for j in range(40)] for i in range(40)])
    for x in range(40):
        ids = np.array([y for y in range(40) if y != x])
        order = ids[np.argsort(rs.batch_scores(x, ids), kind="stable")]
        assert np.array_equal(order, ids[np.argsort(dmat[x, ids], kind="stable")])


def test_kl_batch_consistent_with_subsets(cuda):
    pts = b2.sample_simplex_uniform(10, 300, 8)
    rs = b2.KlRankingSystem(pts)
    rng = np.random.default_rng(0)
    for x in (0, 3, 299):
        full = rs.batch_scores(x)
        ids = rng.choice(300, size=50, replace=False)
        assert np.array_equal(rs.batch_scores(x, ids), full[ids])


def test_kl_rejects_invalid_simplex_by_default(cuda):
    with pytest.raises(ValueError):
        b2.KlRankingSystem(np.array([[0.7, 0.7], [0.5, 0.5]]))


# ---------------------------------------------------------------------------
# EuclideanRankingSystem (similarity.py:119-140)


def test_euclidean_collinear_and_tie_by_id(cuda):
    assert b2.EuclideanRankingSystem(np.array([[0.0], [1.0], [3.0]])).compare(0, 1, 2) < 0
    assert b2.EuclideanRankingSystem(np.array([[0.0], [1.0], [-1.0]])).compare(0, 1, 2) < 0


def test_euclidean_batch_consistent_and_true_order(cuda):
    rng = np.random.default_rng(4)
    vecs = rng.standard_normal((200, 7))
    rs = b2.EuclideanRankingSystem(vecs)
    for x in (0, 42, 199):
        full = rs.batch_scores(x)
        ids = rng.choice(200, size=60, replace=False)
        assert np.array_equal(rs.batch_scores(x, ids), full[ids])
        true = ((vecs - vecs[x]) ** 2).sum(axis=1)
        others = np.array([y for y in range(200) if y != x])
        assert np.array_equal(others[np.argsort(full[others], kind="stable")],
                              others[np.argsort(true[others], kind="stable")])


# ---------------------------------------------------------------------------
# exact_knn / recall (evaluation.py:36-137)


def test_exact_knn_line_points(cuda):
    pts = np.array([[0.0], [1.0], [3.0], [7.0]])
    g = b2.exact_knn(b2.Dataset(pts), b2.EuclideanRankingSystem(pts), 2)
    assert [list(g.of(x)) for x in range(4)] == [[1, 2], [0, 2], [1, 0], [2, 1]]


def test_exact_knn_forced_case_sorts_everything(cuda):
    pts = b2.sample_simplex_uniform(3, 5, 1)
    rs = b2.KlRankingSystem(pts)
    g = b2.exact_knn(b2.Dataset(pts), rs, 4)
    for x in range(5):
        assert list(g.of(x)) == sorted((y for y in range(5) if y != x), key=lambda y: (rs.score(x, y), y))


def test_exact_knn_against_divergence_matrix_argsort(cuda):
    n, k = 200, 8
    pts = b2.sample_simplex_uniform(6, n, 2)
    g = b2.exact_knn(b2.Dataset(pts), b2.KlRankingSystem(pts), k)
    dmat = np.array([[rel_entr(pts[i], pts[j]).sum() for j in range(n)] for i in range(n)])
    np.fill_diagonal(dmat, np.inf)
    for x in range(n):
        assert list(g.of(x)) == list(np.argsort(dmat[x], kind="stable")[:k])


def test_exact_knn_workers_agree_and_rejects_small_n(cuda):
    pts = b2.sample_simplex_uniform(5, 300, 3)
    ds, rs = b2.Dataset(pts), b2.KlRankingSystem(pts)
    assert np.array_equal(b2.exact_knn(ds, rs, 6, workers=1).neighbors, b2.exact_knn(ds, rs, 6, workers=4).neighbors)
    small = b2.sample_simplex_uniform(3, 4, 5)
    with pytest.raises(b2.ConfigError):
        b2.exact_knn(b2.Dataset(small), b2.KlRankingSystem(small), 4)


def test_recall_cases(cuda):
    exact = b2.ExactKnnGraph(np.array([[1, 2], [0, 2], [0, 1]]))
    assert b2.recall(exact.neighbors, exact, [0, 1, 2]) == 1.0
    assert b2.recall(np.array([[3, 4], [3, 4], [3, 4]]), exact, [0, 1, 2]) == 0.0
    assert b2.recall({0: [2, 1], 1: [0, 2], 2: [1, 0]}, exact, [0, 2]) == 1.0
    two = b2.ExactKnnGraph(np.array([[1, 2], [0, 2]]))
    assert b2.recall(np.array([[1, 3], [0, 2]]), two, [0, 1]) == pytest.approx(0.75)
    with pytest.raises(ValueError):
        b2.recall(np.array([[1], [0]]), two, [0])
    with pytest.raises(ValueError):
        b2.recall(np.array([[1], [0]]), b2.ExactKnnGraph(np.array([[1], [0]])), [])
    a, b = b2.uniform_recall_sample(1000, 7), b2.uniform_recall_sample(1000, 7)
    assert np.array_equal(a, b) and a.size == 6 and len(set(map(int, a))) == 6
