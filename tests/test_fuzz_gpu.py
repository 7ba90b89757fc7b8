"""Randomised parity sweep: full descents on the device against the C oracle
(pinned to the reference in tests/test_oracle.py) over seeded random shapes —
n from 60 to 30k, d from 2 to 60, K from 2 to 64, simplex (KL) and Gaussian
(squared Euclidean) data, with the Q23 screen on for part of the KL
cases, and data with duplicated points (exact score ties).  Every round's
table must equal the oracle's exactly (the order contract leaves no freedom:
ties go to the lower id), with the same comparisons, changed rows and FCC
counts, and the same stop round."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2202_00517_b200 as b2
from oracle import native, port
from parity import sha_i32

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(20261021)
    out = []
    for i in range(24):
        k = int(rng.choice([2, 3, 5, 8, 10, 16, 20, 24, 30, 32, 40, 64]))
        n = int(rng.integers(max(3 * k, 60), 30_000))
        d = int(rng.choice([2, 3, 5, 7, 10, 16, 20, 24, 33, 50, 60]))
        metric = "kl" if i % 3 else "l2"
        q23 = i % 2 == 0 and k <= 32  # the Q23 screen rows where the shape has them, else (and odd cases) fp32
        dup = i % 5 == 4
        out.append((i, n, d, k, metric, q23, dup))
    # edge-heavy shapes: tiny K, n barely above K, one- and two-dimensional data
    # (d = 1 KL: every point is 1.0, every score ties), many duplicates
    for j, (n, d, k, metric, q23, dup) in enumerate([
            (7, 3, 2, "kl", True, False), (40, 1, 3, "kl", True, False), (300, 2, 2, "kl", False, True),
            (2000, 12, 2, "kl", True, True), (5000, 20, 3, "kl", True, True), (65, 5, 64, "kl", False, False),
            (3000, 1, 4, "l2", True, False), (4000, 2, 2, "l2", True, True), (20000, 9, 64, "l2", False, True),
            (25000, 16, 32, "kl", True, True), (1200, 60, 64, "kl", False, True), (600, 33, 20, "l2", False, False)]):
        out.append((100 + j, n, d, k, metric, q23, dup))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}_n{c[1]}_d{c[2]}_k{c[3]}_{c[4]}"
                         + ("_q23" if c[5] else "") + ("_dup" if c[6] else ""))
def test_descent_matches_oracle(cuda, monkeypatch, case):
    i, n, d, k, metric, q23, dup = case
    monkeypatch.setenv("KNND_Q23", "1" if q23 else "0")
    rng = np.random.default_rng(1000 + i)
    if metric == "kl":
        pts = port.simplex_points(d, n, rng)
        if dup:  # a block of repeated points: exact fp64 ties everywhere among them
            pts[n // 2: n // 2 + n // 10] = pts[n // 3]
        rs = b2.KlRankingSystem(pts, validate=False)
        tab = native.Tables(pts)
    else:
        pts = rng.normal(size=(n, d)) * rng.uniform(0.5, 3.0) + rng.uniform(-5, 5)
        if dup:
            pts[n // 2: n // 2 + n // 10] = pts[n // 3]
        rs = b2.EuclideanRankingSystem(pts)
        tab = native.L2Tables(pts)
    seed = 7 + i
    cfg = b2.DescentConfig(k=k, seed=seed)
    friends, hist = b2.run(b2.Dataset(pts), rs, cfg)
    init = native.sort_rows(tab, port.random_kout_draws(n, k, port.substream(seed, port.TAG_INIT)))
    shas = []
    final, ohist = native.descend(tab, init, seed, cfg.fcc_sample_count, cfg.resolved_max_rounds(n),
                                  on_round=lambda r, prev, new: shas.append(sha_i32(new)))
    assert [(h.comparisons, h.changed_friend_sets, round(h.fcc * cfg.fcc_sample_count)) for h in hist] == \
        [(h["comparisons"], h["changed"], h["fcc_count"]) for h in ohist]
    assert np.array_equal(friends, final.astype(np.int64))
