"""Host-side logic of the drop-in API (no GPU): config validation, budgets,
RNG substreams and the host draws, which must consume the reference's numpy
streams exactly (checked against the oracle port and the golden fixtures)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2202_00517_b200 as b2
from oracle import port
from paper_2202_00517_b200.engine import Shard
from parity import sha_i32


def test_round_budget_table(known):
    for n, k, b in known["round_budget"]:
        assert b2.round_budget(n, k) == b
    assert b2.round_budget(256, 16) == 4 and b2.round_budget(16, 16) == 2
    with pytest.raises(b2.ConfigError):
        b2.round_budget(1, 16)
    with pytest.raises(b2.ConfigError):
        b2.round_budget(100, 1)


def test_descent_config_validation():
    cfg = b2.DescentConfig(k=16)
    assert cfg.fcc_sample_count == 1000 and cfg.resolved_workers() == 1
    assert cfg.resolved_max_rounds(20_000) == b2.round_budget(20_000, 16) + 4
    assert b2.DescentConfig(k=4, max_rounds=3).resolved_max_rounds(10_000) == 3
    assert b2.DescentConfig(k=4, worker_count="auto").resolved_workers() >= 1
    for bad in (dict(k=1), dict(k=4, fcc_sample_count=0), dict(k=4, max_rounds=0), dict(k=4, worker_count=0),
                dict(k=4, worker_count="many")):
        with pytest.raises(b2.ConfigError):
            b2.DescentConfig(**bad)
    assert issubclass(b2.ConfigError, ValueError)


def test_dataset_and_ranking_validation():
    with pytest.raises(b2.ConfigError):
        b2.Dataset(np.zeros((1, 3)))
    with pytest.raises(ValueError):
        b2.KlRankingSystem(np.array([[0.6, 0.6]]))
    with pytest.raises(ValueError):
        b2.KlRankingSystem(np.array([[0.5, 0.0, 0.5]]))
    b2.KlRankingSystem(np.array([[0.6, 0.6]]), validate=False)
    with pytest.raises(ValueError):
        b2.sample_simplex_uniform(1, 10, 0)
    with pytest.raises(ValueError):
        b2.sample_simplex_uniform(3, 0, 0)


def test_derive_rng_substreams():
    a = b2.derive_rng(5, 3, 1).integers(0, 1 << 32, 8)
    assert np.array_equal(a, b2.derive_rng(5, 3, 1).integers(0, 1 << 32, 8))
    assert not np.array_equal(a, b2.derive_rng(5, 3, 2).integers(0, 1 << 32, 8))
    assert not np.array_equal(a, b2.derive_rng(6, 3, 1).integers(0, 1 << 32, 8))
    assert b2.derive_rng(-1, 2).integers(0, 10) in range(10)
    assert np.array_equal(b2.derive_rng(7, 1, 20).integers(0, 99, 5), port.substream(7, 1, 20).integers(0, 99, 5))


@pytest.mark.parametrize("n,d,seed", [(300, 6, 3), (2000, 20, 0), (100_000, 10, 0)])
def test_points_generator_matches_reference_stream(n, d, seed):
    a = b2.sample_simplex_uniform(d, n, b2.derive_rng(seed, b2.STREAM_DATA, d))
    assert np.array_equal(a, port.experiment_points(n, d, seed))


@pytest.mark.parametrize("n,k", [(300, 7), (5, 4), (12, 6), (800, 40), (100_000, 20), (20_000, 3)])
def test_random_kout_draws_consume_the_reference_stream(n, k):
    a = b2.random_kout_draws(n, k, b2.derive_rng(11, 2))
    b = port.random_kout_draws(n, k, port.substream(11, 2))
    assert np.array_equal(a, b)
    anchors = np.arange(n)[:, None]
    assert not (a == anchors).any()
    s = np.sort(a, axis=1)
    assert not (s[:, 1:] == s[:, :-1]).any()


def test_rejection_redraws_are_exercised():
    # n - 1 > 2K^2 but small enough that first draws collide in some rows
    n, k = 60, 5
    rng = b2.derive_rng(3, 2)
    first = rng.integers(0, n - 1, size=(n, k), dtype=np.int64)
    first += first >= np.arange(n)[:, None]
    s = np.sort(first, axis=1)
    assert (s[:, 1:] == s[:, :-1]).any(), "the seed must produce at least one redraw"
    assert np.array_equal(b2.random_kout_draws(n, k, b2.derive_rng(3, 2)), port.random_kout_draws(n, k, port.substream(3, 2)))


@pytest.mark.parametrize("r", [1, 2, 7])
def test_fcc_samples_match_reference_stream(r):
    got = b2.fcc_samples(1000, 20, 1000, b2.derive_rng(0, 3, r))
    xs, i, j = port.fcc_draws(1000, 20, 1000, port.substream(0, 3, r))
    assert np.array_equal(got, np.stack([xs, i, j]).astype(np.int32))
    assert (got[1] != got[2]).all()


def test_fcc_schedule_is_round_indexed():
    cfg = b2.DescentConfig(k=10, seed=4)
    from paper_2202_00517_b200.descent import draw_fcc_schedule

    sched = draw_fcc_schedule(5000, 10, cfg, 6)
    for r in range(1, 7):
        assert np.array_equal(sched[r - 1], b2.fcc_samples(5000, 10, 1000, b2.derive_rng(4, 3, r)))


def test_fcc_schedule_draws_chunks_on_demand():
    """FccSchedule (what run() uses) gives every round the sample of the
    up-front schedule, drawing only the chunks the rounds reach."""
    import torch

    from paper_2202_00517_b200.descent import FccSchedule, draw_fcc_schedule

    cfg = b2.DescentConfig(k=10, seed=4)
    full = draw_fcc_schedule(5000, 10, cfg, 11)
    sched = FccSchedule(5000, 10, cfg, 11, torch.device("cpu"))
    assert len(sched) == 11 and not sched._chunks
    for r in (1, 2, 5, 9, 11):
        assert np.array_equal(sched[r - 1].numpy(), full[r - 1])
    assert list(sched._chunks) == [2]  # only the last chunk touched is kept
    with pytest.raises(IndexError):
        sched[11]


def test_k_above_device_limit_is_a_config_error():
    b2.DescentConfig(k=64)
    with pytest.raises(b2.ConfigError, match="<= 64"):
        b2.DescentConfig(k=65)


def test_batch_score_ids_index_like_numpy():
    """ids of batch_scores follow numpy indexing (the reference's self._log[ids]):
    negative ids wrap, out-of-range ids raise IndexError, masks select."""
    from paper_2202_00517_b200.similarity import _index_ids

    n = 10
    ref = np.arange(n)
    for ids in ([0, 9, -1, -10], np.array([3, -3], dtype=np.int16), [], np.arange(n) % 2 == 0):
        x, got = _index_ids(-2, ids, n)
        assert x == 8 and got.dtype == np.int32
        assert np.array_equal(got, ref[np.asarray(ids, dtype=None if len(ids) else np.int64)])
    assert np.array_equal(_index_ids(3, None, n)[1], ref)
    for bad in ([10], [-11], [0, 2**40]):
        with pytest.raises(IndexError):
            _index_ids(0, bad, n)
        with pytest.raises(IndexError):
            ref[np.asarray(bad)]
    for badx in (10, -11):
        with pytest.raises(IndexError):
            _index_ids(badx, [0], n)
    with pytest.raises(IndexError):
        _index_ids(0, np.array([0.5]), n)


@pytest.mark.parametrize("n,world", [(10, 1), (10, 3), (1_000_000, 8), (7, 8), (100_001, 2)])
def test_shards_cover_rows_once(n, world):
    shards = [Shard(r, world, n) for r in range(world)]
    covered = np.zeros(n, dtype=int)
    for s in shards:
        assert s.padded_rows >= n and s.padded_rows == s.chunk * world
        covered[s.lo:s.hi] += 1
        assert s.hi - s.lo <= s.chunk
    assert (covered == 1).all()


def test_golden_init_is_reachable_from_host_draws(small_meta, small_tables):
    """The host draws + the oracle row sort reproduce the reference's initial table,
    so the device only has to reproduce the row sort."""
    from oracle import native

    for name in ("n300_d6_k7_s3", "n1000_d20_k20_s1"):
        meta = small_meta[name]
        pts = b2.sample_simplex_uniform(meta["d"], meta["n"], b2.derive_rng(meta["seed"], 1, meta["d"]))
        draws = b2.random_kout_draws(meta["n"], meta["k"], b2.derive_rng(meta["seed"], 2))
        assert sha_i32(native.sort_rows(native.Tables(pts), draws)) == meta["init_sha"]


# ---------------------------------------------------------------------------
# host helpers of the API (similarity.py:36-47, core.py:196-235)


def test_kl_divergence_helper():
    from scipy.special import rel_entr

    x, y = np.array([0.5, 0.5]), np.array([0.25, 0.75])
    assert b2.kl_divergence(x, y) == pytest.approx(0.143841, abs=1e-6)
    assert b2.kl_divergence(y, x) == pytest.approx(0.130812, abs=1e-6)
    assert b2.kl_divergence(x, x) == 0.0
    rng = np.random.default_rng(1)
    for _ in range(20):
        e = rng.standard_exponential((2, 8))
        p, q = e / e.sum(axis=1, keepdims=True)
        assert b2.kl_divergence(p, q) == pytest.approx(float(rel_entr(p, q).sum()), rel=1e-12)
    with pytest.raises(ValueError):
        b2.kl_divergence(np.array([0.5, 0.5]), np.array([0.2, 0.3, 0.5]))
    with pytest.raises(ValueError):
        b2.kl_divergence(np.array([0.0, 1.0]), np.array([0.5, 0.5]))


def test_build_cofriends():
    assert b2.build_cofriends({0: {1}, 1: {0}}) == {0: {1}, 1: {0}}
    assert b2.build_cofriends({0: {1}, 1: {2}, 2: {0}}) == {1: {0}, 2: {1}, 0: {2}}
    rng = np.random.default_rng(7)
    friends = {x: set(map(int, (lambda r: r + (r >= x))(rng.permutation(99)[:5]))) for x in range(100)}
    cof = b2.build_cofriends(friends)
    for y in range(100):
        assert cof[y] == {x for x in range(100) if y in friends[x]}


class _LineRanking(b2.RankingSystem):
    """Points on a line ranked by distance, ties by id (host-only, for the checker)."""

    def __init__(self, pos):
        self.pos = pos

    def compare(self, x, y, z):
        return -1 if (abs(self.pos[y] - self.pos[x]), y) < (abs(self.pos[z] - self.pos[x]), z) else 1


class _Cyclic(b2.RankingSystem):
    def compare(self, x, y, z):  # y < z iff (z - y) mod 3 == 1: intransitive on {0, 1, 2}
        return -1 if (z - y) % 3 == 1 else 1


def test_verify_total_order():
    rs = _LineRanking([0.0, 1.0, -1.0, 3.0, 2.5])
    assert b2.verify_total_order(rs, 0, range(5))
    assert not b2.verify_total_order(_Cyclic(), 5, [0, 1, 2])


def test_fused_exchange_states_never_alias_a_reused_table(small_meta):
    """The ping-pong tables of the fused exchange are reused every other round
    (and by the next descent): a state handed to on_round raises once a later
    round has overwritten its table (instead of silently showing another
    table), and the final state is a private copy (engine.PeerTables.gen,
    KnnState._detach)."""
    import torch

    from cpu_ops import CpuOps
    from oracle import native
    from paper_2202_00517_b200.descent import descend_resident, draw_fcc_schedule
    from paper_2202_00517_b200.engine import Engine, PeerTables

    meta = small_meta["n1000_d20_k20_s1"]
    n, d, k, seed = meta["n"], meta["d"], meta["k"], meta["seed"]
    pts = b2.sample_simplex_uniform(d, n, b2.derive_rng(seed, 1, d))
    cfg = b2.DescentConfig(k=k, seed=seed)
    rounds = cfg.resolved_max_rounds(n)
    eng = Engine(n, k, torch.device("cpu"), ops=CpuOps())
    bufs = [eng.alloc_table() for _ in range(2)]
    assert eng.enable_peer_exchange(PeerTables(bufs, [[], []], lambda i: None))
    table = eng.alloc_table()
    eng.upload_rows(b2.random_kout_draws(n, k, b2.derive_rng(seed, 2)), table)
    seen = []
    state, hist = descend_resident(eng, native.Tables(pts), table, torch.from_numpy(draw_fcc_schedule(n, k, cfg, rounds)),
                                   cfg.fcc_sample_count, rounds, on_round=lambda st, s: seen.append(st))
    assert sha_i32(state.friends) == meta["rounds"][-1]["sha"]
    assert all(state._table.data_ptr() != b.data_ptr() for b in bufs)  # the final table is private
    assert len(seen) == len(hist) >= 3
    seen[-1]._table  # the last round's table was not reused
    for st in seen[:-2]:  # tables overwritten two rounds later
        with pytest.raises(RuntimeError, match="reused by a later round"):
            st.friends


def test_q23_row_sizes():
    """3 bytes per entry in the smallest row the kernels have; none where it would not pay."""
    from paper_2202_00517_b200.similarity import q23_row_bytes

    assert [q23_row_bytes(d) for d in (1, 5, 6, 10, 11, 16, 17, 20, 21)] == [16, 16, 32, 32, 48, 48, 64, 64, 64]
    assert [q23_row_bytes(d) for d in (22, 42, 43, 50, 53, 54, 96)] == [0, 0, 160, 160, 160, 0, 0]
