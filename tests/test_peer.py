"""The fused join + table exchange (knnd_local_join_peers, engine.PeerTables)
on one B200.  Only one GPU is available to these tests, so the peer tables are
extra buffers on the same device: the kernel's multi-destination row stores,
the ping-pong table logic and the barrier placement are what is checked here;
the multi-rank logic is covered under gloo in test_multirank.py, and the
symmetric-memory mapping itself at world size 1."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2202_00517_b200 as b2
from oracle import port
from parity import sha_i32
from paper_2202_00517_b200.engine import Csr, Engine, PeerTables

pytestmark = pytest.mark.gpu

NAME = "n1000_d20_k20_s1"


def _case(small_meta, name=NAME):
    meta = small_meta[name]
    return meta, port.experiment_points(meta["n"], meta["d"], meta["seed"])


@pytest.mark.parametrize("metric", ["kl", "l2"])
@pytest.mark.parametrize("npeers", [1, 3, 15])
def test_join_stores_rows_into_every_peer_table(cuda, small_meta, small_tables, metric, npeers):
    """Rows of a partial anchor range [lo, hi) land at rows lo..hi-1 of every
    peer table (absolute row ids), identical to out_ids; nothing else is touched."""
    meta, pts = _case(small_meta)
    n, k = meta["n"], meta["k"]
    rs = b2.KlRankingSystem(pts, validate=False) if metric == "kl" else b2.EuclideanRankingSystem(pts)
    st = b2.KnnState(small_tables[f"{NAME}/init"])
    tabs = rs.device_tables()
    lo, hi = 137, 811
    csr = Csr(st._csr.indptr[lo:hi + 1] - st._csr.indptr[lo], st._csr.indices[int(st._csr.indptr[lo]):], lo, hi)
    ref = torch.empty((hi - lo, k), dtype=torch.int32, device=cuda)
    tally = torch.zeros(4, dtype=torch.int64, device=cuda)
    st._engine.ops.join(tabs, st._table, n, k, csr, st._max_indeg, ref, tally)
    peers = [torch.full((n, k), -5, dtype=torch.int32, device=cuda) for _ in range(npeers)]
    out = torch.empty_like(ref)
    tally2 = torch.zeros(4, dtype=torch.int64, device=cuda)
    st._engine.ops.join(tabs, st._table, n, k, csr, st._max_indeg, out, tally2,
                        peers=[t.data_ptr() for t in peers])
    assert torch.equal(out, ref) and torch.equal(tally, tally2)
    for t in peers:
        assert torch.equal(t[lo:hi], ref)
        assert bool((t[:lo] == -5).all()) and bool((t[hi:] == -5).all())


def test_peer_count_is_validated(cuda, small_meta, small_tables):
    meta, pts = _case(small_meta)
    st = b2.KnnState(small_tables[f"{NAME}/init"])
    rs = b2.KlRankingSystem(pts, validate=False)
    out = torch.empty((meta["n"], meta["k"]), dtype=torch.int32, device=cuda)
    tally = torch.zeros(4, dtype=torch.int64, device=cuda)
    with pytest.raises(b2.KnndError, match="npeers"):
        st._engine.ops.join(rs.device_tables(), st._table, meta["n"], meta["k"], st._csr, st._max_indeg, out,
                            tally, peers=[out.data_ptr()] * 16)


def test_engine_fused_exchange_trajectory(cuda, small_meta, small_tables):
    """A full descent with the engine in fused-exchange mode (ping-pong tables,
    one mirror per table standing in for a peer): the reference trajectory,
    and after every round the mirror of the written table equals it."""
    from paper_2202_00517_b200.descent import descend_resident, draw_fcc_schedule, _to_device

    meta, pts = _case(small_meta)
    n, k, seed = meta["n"], meta["k"], meta["seed"]
    rs = b2.KlRankingSystem(pts, validate=False)
    cfg = b2.DescentConfig(k=k, seed=seed)
    eng = Engine(n, k, cuda)
    bufs = [eng.alloc_table() for _ in range(2)]
    mirrors = [eng.alloc_table().fill_(-1) for _ in range(2)]
    barriers = []
    eng.enable_peer_exchange(PeerTables(bufs, [[mirrors[0].data_ptr()], [mirrors[1].data_ptr()]],
                                        lambda i: barriers.append(i)))
    table = eng.alloc_table()
    eng.upload_rows(b2.random_kout_draws(n, k, b2.derive_rng(seed, 2)), table)
    rounds = cfg.resolved_max_rounds(n)
    smp = _to_device(draw_fcc_schedule(n, k, cfg, rounds), cuda)
    seen = []

    def check(state, stats):
        i = 0 if state._table.data_ptr() == bufs[0].data_ptr() else 1
        assert state._table.data_ptr() == bufs[i].data_ptr()
        assert torch.equal(mirrors[i][:n], bufs[i][:n])
        seen.append(i)

    state, hist = descend_resident(eng, rs.device_tables(), table, smp, cfg.fcc_sample_count, rounds,
                                   on_round=check)
    expect = [(r["comparisons"], r["changed"], r["fcc"]) for r in meta["rounds"]]
    assert [(h.comparisons, h.changed_friend_sets, h.fcc) for h in hist] == expect
    assert sha_i32(state.friends) == meta["rounds"][-1]["sha"]
    assert seen == [r % 2 for r in range(len(hist))]  # round 1 writes table 0, then alternate
    assert barriers == []  # world size 1: no cross-rank barrier


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_symmetric_peer_tables_world1(cuda):
    """torch symmetric memory maps the ping-pong tables (world size 1 under NCCL):
    the rendezvous, buffer addresses and the device barrier work on this box."""
    from paper_2202_00517_b200.engine import symmetric_peer_tables

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        eng = Engine(1000, 20, cuda)
        pt = symmetric_peer_tables(eng)
        assert [b.shape for b in pt.bufs] == [(1000, 20), (1000, 20)]
        assert pt.peers == [[], []]
        assert symmetric_peer_tables(Engine(1000, 20, cuda)) is pt  # one mapping per shape and group
        pt.bufs[0].fill_(3)
        pt.barrier(0)
        pt.barrier(1)
        torch.cuda.synchronize()
        assert int(pt.bufs[0].sum()) == 3 * 20000
    finally:
        dist.destroy_process_group()
