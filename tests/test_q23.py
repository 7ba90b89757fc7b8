"""The join's 23-bit fixed-point screen (knnd_kl_q23_prepare + the q23 path of
knnd_local_join_peers: 3 bytes per entry, 64-byte rows at d = 20; on by
default for d <= 21, K <= 32) and the fp32 screen it replaces (KNND_Q23=0).
Either screen only prunes candidates (with a rigorous error bound) and orders
certified rows; the fp64 decision is unchanged, so every table must equal the
reference's / the oracle's exactly with both."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import paper_2202_00517_b200 as b2
from oracle import native, port
from parity import sha_i32

pytestmark = pytest.mark.gpu


@pytest.fixture
def q23_on(monkeypatch):
    monkeypatch.setenv("KNND_Q23", "1")


@pytest.fixture(params=["q23", "fp32"])
def screen(request, monkeypatch):
    monkeypatch.setenv("KNND_Q23", "1" if request.param == "q23" else "0")
    return request.param


def test_q23_table_quantisation(cuda, q23_on):
    """q = round((Lmax_j - log) / h_j) per column in 3 little-endian bytes at
    byte 3 j of a 64-byte row; Lmax_j - h_j q is within h_j / 2 of the fp64 log."""
    pts = port.experiment_points(5000, 20, 1)
    tabs = b2.KlRankingSystem(pts, validate=False).device_tables()
    assert tabs.q23 is not None and tabs.q23_bytes == 64
    raw = tabs.q23.cpu().numpy()
    assert (raw[:, 60:] == 0).all()
    b = raw[:, :60].reshape(-1, 20, 3).astype(np.int64)
    q = (b[..., 0] | (b[..., 1] << 8) | (b[..., 2] << 16)).astype(np.float64)
    assert q.max() <= 2 ** 23 - 1
    h = tabs.qh23.cpu().numpy().astype(np.float64)
    lg = np.log(pts)
    lo, hi = lg.min(axis=0), lg.max(axis=0)
    hd = (hi - lo) / (2 ** 23 - 1)
    np.testing.assert_allclose(h[:20], hd, rtol=1e-6)
    assert (h[20:] == 0).all()
    err = np.abs(hi - hd * q - lg)
    assert (err <= hd / 2 * (1 + 1e-6)).all()


def test_q23_non_finite_logs_keep_fp32(cuda, q23_on):
    """A zero coordinate (log = -inf) cannot be quantised: the tables keep the fp32 screen."""
    pts = port.experiment_points(500, 8, 2).copy()
    pts[3, 2] = 0.0
    tabs = b2.KlRankingSystem(pts, validate=False).device_tables()
    assert tabs.q23 is None


@pytest.mark.parametrize("name", ["n1000_d20_k20_s1", "n1500_d16_k10_s7", "n800_d10_k40_s5", "n600_d50_k30_s2",
                                  "n4000_d5_k10_s0"])
def test_q23_small_trajectories(cuda, screen, small_meta, name):
    """Full descents with the q23 screen reproduce the reference's per-round
    tables (d = 20, 16, 10, 50, 5: rows of 64 / 48 / 32 / 160 / 16 bytes; K = 40 > 32 takes
    the fp32 screen)."""
    meta = small_meta[name]
    n, d, k, seed = meta["n"], meta["d"], meta["k"], meta["seed"]
    pts = port.experiment_points(n, d, seed)
    rs = b2.KlRankingSystem(pts, validate=False)
    friends, hist = b2.run(b2.Dataset(pts), rs, b2.DescentConfig(k=k, seed=seed))
    assert [(h.comparisons, h.changed_friend_sets, round(h.fcc * 1000)) for h in hist] == \
        [(r["comparisons"], r["changed"], r["fcc_count"]) for r in meta["rounds"]]
    assert sha_i32(friends) == meta["rounds"][-1]["sha"]


def test_q23_c2_trajectory(cuda, screen, trajectories):
    """C2 (n = 100k, d = 10, K = 20) with the q23 screen: every round's table sha,
    comparisons, changed rows and FCC count equal the reference's."""
    ref = trajectories["c2"]
    n, d, k, seed = ref["n"], ref["d"], ref["k"], ref["seed"]
    pts = port.experiment_points(n, d, seed)
    rs = b2.KlRankingSystem(pts, validate=False)
    assert (rs.device_tables().q23 is not None) == (screen == "q23")
    cfg = b2.DescentConfig(k=k, seed=seed)
    st = b2.init_random_kout(b2.Dataset(pts), rs, cfg, b2.derive_rng(seed, 2))
    for r in ref["rounds"]:
        st, stats = b2.run_round(st, rs, cfg)
        assert sha_i32(st.friends) == r["sha"], r["round"]
        assert (stats.comparisons, stats.changed_friend_sets, round(stats.fcc * 1000)) == \
            (r["comparisons"], r["changed"], r["fcc_count"])


def test_q23_size_classes_and_hubs_vs_oracle(cuda, screen):
    """Every size class (warp, 128/256/512-thread blocks, global-memory hubs)
    through the q23 screen: rows and |U| equal the C oracle's."""
    from test_gpu import _hub_table

    n, d, k = 30000, 20, 20
    rng = np.random.default_rng(n + d + k)
    pts = port.experiment_points(n, d, 3)
    hubs = [(7, n // 4), (11, n // 10), (13, 40 * k), (17, 8 * k), (19, 3 * k), (23, 2 * k)]
    table = native.sort_rows(native.Tables(pts), _hub_table(n, k, hubs, rng))
    rs = b2.KlRankingSystem(pts, validate=False)
    st = b2.KnnState(table)
    tabs = rs.device_tables()
    assert (tabs.q23 is not None) == (screen == "q23")
    out = torch.empty((n, k), dtype=torch.int32, device=cuda)
    uc = torch.empty(n, dtype=torch.int32, device=cuda)
    tally = torch.zeros(4, dtype=torch.int64, device=cuda)
    st._engine.ops.join(tabs, st._table, n, k, st._csr, st._max_indeg, out, tally, None, uc)
    o_rows, _, o_uc, o_comp, o_changed = native.local_join(native.Tables(pts), table)
    assert np.array_equal(uc.cpu().numpy(), o_uc)
    assert np.array_equal(out.cpu().numpy(), o_rows)
    assert tally.cpu().tolist()[:3] == [o_comp, o_changed, 0]


def test_q23_unnormalised_scales_keep_fp32_rows(cuda, q23_on):
    """The screen's fp32 weights x_j h_j 2^126 must stay in the normal range: KL data far
    from the simplex (validate=False) screen the fp32 rows, and a round still equals the oracle's."""
    base = port.experiment_points(1500, 8, 4)
    for scale, q23 in ((1.0, True), (3.0, True), (1e7, False)):
        pts = base * scale
        rs = b2.KlRankingSystem(pts, validate=False)
        assert (rs.device_tables().q23 is not None) == q23, scale
        k = 10
        tab = native.Tables(pts)
        init = native.sort_rows(tab, port.random_kout_draws(1500, k, port.substream(3, port.TAG_INIT)))
        nxt, s = b2.run_round(b2.KnnState(init), rs, b2.DescentConfig(k=k, seed=3))
        rows, _, _, comps, changed = native.local_join(tab, init)
        assert np.array_equal(nxt.friends, rows), scale
        assert (s.comparisons, s.changed_friend_sets) == (comps, changed)
