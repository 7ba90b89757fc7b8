"""Row-sharded rounds over 1 and 2 ranks (gloo, CPU): the sharding, the
in-place table all-gather and the tally all-reduce of engine.py give the
reference's trajectory bit for bit, whatever the rank count (the GPU analogue
of t_descent:232-242, worker counts agree)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

NAME = "n1000_d20_k20_s1"


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, meta, out, shared=None):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2202_00517_b200 as b2
    from cpu_ops import CpuOps
    from oracle import native
    from paper_2202_00517_b200.descent import descend_resident, draw_fcc_schedule
    from paper_2202_00517_b200.engine import Engine
    from parity import sha_i32

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, d, k, seed = meta["n"], meta["d"], meta["k"], meta["seed"]
        pts = b2.sample_simplex_uniform(d, n, b2.derive_rng(seed, 1, d))
        tab = native.Tables(pts)
        cfg = b2.DescentConfig(k=k, seed=seed)
        rounds = cfg.resolved_max_rounds(n)
        eng = Engine(n, k, torch.device("cpu"), ops=CpuOps())
        assert eng.shard.world == world and eng.shard.rank == rank
        if shared is not None:  # fused exchange: every rank's ping-pong tables in shared memory
            from paper_2202_00517_b200.engine import PeerTables

            peers = [[shared[q][i] for q in range(world) if q != rank] for i in range(2)]
            assert eng.enable_peer_exchange(PeerTables(shared[rank], peers, lambda i: dist.barrier()))
        table = eng.alloc_table()
        eng.upload_rows(b2.random_kout_draws(n, k, b2.derive_rng(seed, 2)), table)
        smp = torch.from_numpy(draw_fcc_schedule(n, k, cfg, rounds))
        state, hist = descend_resident(eng, tab, table, smp, cfg.fcc_sample_count, rounds)
        if shared is not None:
            assert state._table.data_ptr() not in (shared[rank][0].data_ptr(), shared[rank][1].data_ptr())  # a private copy
        out[rank] = {"sha": sha_i32(state.friends),
                     "hist": [(h.comparisons, h.changed_friend_sets, h.fcc) for h in hist]}
    finally:
        dist.destroy_process_group()


def _run(world, meta, peer=False):
    mgr = mp.Manager()
    out = mgr.dict()
    shared = None
    if peer:
        rows = -(-meta["n"] // world) * world
        shared = [[torch.full((rows, meta["k"]), -7, dtype=torch.int32).share_memory_() for _ in range(2)]
                  for _ in range(world)]
    mp.spawn(_worker, args=(world, _free_port(), meta, out, shared), nprocs=world, join=True)
    return dict(out)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_rounds_match_reference(small_meta, world):
    meta = small_meta[NAME]
    res = _run(world, meta)
    expect = [(r["comparisons"], r["changed"], r["fcc"]) for r in meta["rounds"]]
    for rank in range(world):
        assert res[rank]["hist"] == expect, rank
        assert res[rank]["sha"] == meta["rounds"][-1]["sha"], rank


@pytest.mark.parametrize("world", [2, 3])
def test_fused_peer_exchange_matches_reference(small_meta, world):
    """The fused exchange (engine.PeerTables, each rank's join storing its rows
    into every peer's copy, a barrier instead of the all-gather) on shared-memory
    tables: same trajectory and final table as the reference."""
    meta = small_meta[NAME]
    res = _run(world, meta, peer=True)
    expect = [(r["comparisons"], r["changed"], r["fcc"]) for r in meta["rounds"]]
    for rank in range(world):
        assert res[rank]["hist"] == expect, rank
        assert res[rank]["sha"] == meta["rounds"][-1]["sha"], rank


def _consensus_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2202_00517_b200 import engine as E

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def mapped(eng):  # rank 1 cannot map the peer tables, rank 0 can
            if eng.shard.rank == 1:
                raise RuntimeError("no peer access")
            return E.PeerTables([eng.alloc_table(), eng.alloc_table()], [[], []], lambda i: None)

        E.exchange_mode = lambda eng: "peer"
        E.peer_capable = lambda eng: True
        E.symmetric_peer_tables = mapped
        eng = E.Engine(100, 4, torch.device("cpu"), ops=object())
        out[rank] = (eng.enable_peer_exchange(), eng.peer is None)
    finally:
        dist.destroy_process_group()


def test_peer_exchange_fallback_is_collective():
    """If any rank fails to map the symmetric tables, every rank falls back to
    the all-gather (mixed exchanges would deadlock the rounds)."""
    out = mp.Manager().dict()
    mp.spawn(_consensus_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert dict(out) == {0: (False, True), 1: (False, True)}
