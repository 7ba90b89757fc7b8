"""The row-sharded, fused-exchange path with the real CUDA kernels, 2, 3, 4
and 8 ranks as processes sharing one GPU (P = 1, 2, 4, 8 agree).

Each rank is its own process on cuda:0 with its own copy of the tables.  The
two ping-pong next tables of every rank are exported with CUDA IPC and opened
by the other ranks (the same mapping torch symmetric memory makes across
GPUs), so knnd_local_join_peers stores each finished row into every rank's
copy exactly as on a multi-GPU node.  The cross-rank barrier is a host one
(stream synchronise, then a gloo barrier), and the tally all-reduce goes
through gloo: no kernel ever waits on another process's kernel, so sharing
one GPU cannot deadlock (B200_PROFILING.md: ranks whose kernels wait on each
other must not share a GPU).  The reference's own guarantee is worker-count
independence (descent.py:292-302): every rank must reproduce the
reference trajectory (comparisons, changed rows, FCC per round) and its final
table, for any rank count.
"""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _open_peer(handle, numel):
    storage = torch.UntypedStorage._new_shared_cuda(*handle)
    t = torch.empty(0, dtype=torch.int32, device="cuda")
    t.set_(storage, 0, (numel,), (1,))
    return t


def _worker(rank, world, port, case, out):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import paper_2202_00517_b200 as b2
    from paper_2202_00517_b200.descent import FccSchedule, descend_resident
    from paper_2202_00517_b200.engine import Engine, PeerTables
    from parity import sha_i32

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        n, d, k, seed = case["n"], case["d"], case["k"], case["seed"]
        pts = b2.sample_simplex_uniform(d, n, b2.derive_rng(seed, 1, d))
        rs = b2.KlRankingSystem(pts, validate=False)
        cfg = b2.DescentConfig(k=k, seed=seed)
        rounds = cfg.resolved_max_rounds(n)
        eng = Engine(n, k, dev)
        assert eng.shard.world == world and eng.shard.rank == rank
        # this rank's ping-pong tables, exported over CUDA IPC; the other ranks' opened
        bufs = [eng.alloc_table().fill_(-7) for _ in range(2)]
        torch.cuda.synchronize()
        handles = [b.untyped_storage()._share_cuda_() for b in bufs]
        every = [None] * world
        dist.all_gather_object(every, handles)
        opened = [[_open_peer(every[q][i], bufs[i].numel()) for q in range(world) if q != rank] for i in range(2)]
        peers = [[t.data_ptr() for t in opened[i]] for i in range(2)]

        def barrier(i):
            torch.cuda.current_stream().synchronize()  # this rank's rows are in every copy
            dist.barrier()                             # ... and every other rank's in ours

        assert eng.enable_peer_exchange(PeerTables(bufs, peers, barrier))
        table = eng.alloc_table()
        eng.upload_rows(b2.random_kout_draws(n, k, b2.derive_rng(seed, 2)), table)
        smp = FccSchedule(n, k, cfg, rounds, dev)
        seen = []

        def check(state, stats):
            # after the barrier every copy of the written table holds all rows
            i = eng.peer.index_of(state._table)
            seen.append(sha_i32(bufs[i][:n].cpu().numpy()))

        state, hist = descend_resident(eng, rs.device_tables(), table, smp, cfg.fcc_sample_count, rounds,
                                       on_round=check)
        out[rank] = {"sha": sha_i32(state.friends), "round_shas": seen,
                     "hist": [(h.comparisons, h.changed_friend_sets, h.fcc) for h in hist],
                     "launches": b2.launch_count()}
        dist.barrier()  # keep the exported tables alive until every rank is done reading
        del opened
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True,
                       start_method="spawn")
    return dict(out)


def _expect(meta):
    return [(r["comparisons"], r["changed"], r["fcc"]) for r in meta["rounds"]]


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_fused_exchange_small_case(cuda, small_meta, world):
    meta = small_meta["n1000_d20_k20_s1"]
    res = _run(world, meta)
    for rank in range(world):
        assert res[rank]["hist"] == _expect(meta), rank
        assert res[rank]["round_shas"] == [r["sha"] for r in meta["rounds"]], rank
        assert res[rank]["sha"] == meta["rounds"][-1]["sha"], rank
        assert res[rank]["launches"] > 0


@pytest.mark.parametrize("world", [2, 3, 8])
def test_fused_exchange_c2_trajectory(cuda, trajectories, world):
    """C2 (n = 100k, d = 10, K = 20): every round's table on every rank equals the
    reference's recorded table (sha256), with the reference's tallies."""
    meta = trajectories["c2"]
    res = _run(world, meta)
    for rank in range(world):
        assert res[rank]["hist"] == _expect(meta), rank
        assert res[rank]["round_shas"] == [r["sha"] for r in meta["rounds"]], rank
        assert res[rank]["sha"] == meta["rounds"][-1]["sha"], rank
