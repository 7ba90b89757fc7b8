"""Projected strong scaling of the row-sharded descent from ONE GPU.

Only one B200 is available to this build, so the P-rank timing is
reconstructed: along the C3 trajectory (the real single-GPU rounds), every
round's input is also processed as each rank r of P would — the co-friend CSR
of its own targets and the local join of its own anchors, timed with CUDA
events one shard at a time — and the per-round critical path is the slowest
shard's CSR + join, plus the replicated FCC.  The exchange is the fused peer
store (overlapped with the join) and a device barrier + 32-byte all-reduce,
added as a fixed per-round cost (`--sync-us`, default 30 us), and every P
pays the per-round host cost (`--host-us`, default 80 us, tools/round_overhead.py) less the part
of it that overlaps the CSR build's tail: the round's statistics are read behind an event recorded
inside the build (knnd_csr_build_ev), so only max(0, host - tail) is exposed, the tail (scan + fill)
being timed per shard.  Prints one JSON line per P with the projected descent time and speed-up
over P = 1.

Usage: python tools/shard_projection.py [n d k] [--sync-us 30]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_00517_b200 as b2  # noqa: E402
from paper_2202_00517_b200.engine import Shard  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("n", type=int, nargs="?", default=1_000_000)
ap.add_argument("d", type=int, nargs="?", default=20)
ap.add_argument("k", type=int, nargs="?", default=20)
ap.add_argument("--sync-us", type=float, default=30.0)
# the per-round host cost every P pays (launch sequence, Python, the stats read):
# tools/round_overhead.py measures ~0.23 ms of wall per round at n = 1000, of which
# ~0.15 ms is the tiny kernels' own GPU time (already in the timed CSR / join here)
ap.add_argument("--host-us", type=float, default=80.0)
ap.add_argument("--ranks", default="1,2,4,8")
args = ap.parse_args()
n, d, k = args.n, args.d, args.k
P_LIST = [int(x) for x in args.ranks.split(",")]

dev = torch.device("cuda", 0)
pts = b2.sample_simplex_uniform(d, n, b2.derive_rng(0, b2.STREAM_DATA, d))
rs = b2.KlRankingSystem(pts, validate=False)
tabs = rs.device_tables(dev)
cfg = b2.DescentConfig(k=k, seed=0)


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


def shard_costs(state, P, samples):
    """(max over ranks of CSR ms, max over ranks of join ms, fcc ms) for one round input."""
    eng = state._engine
    csr_ms, join_ms, tails = [], [], []
    for r in range(P):
        s = Shard(r, P, n)
        mx = torch.zeros(2, dtype=torch.int32, device=dev)
        eng.ops.csr(state._table, n, k, s.lo, s.hi, mx[0:1])  # warm (workspace, first launch)
        t_csr = min(timed(lambda: eng.ops.csr(state._table, n, k, s.lo, s.hi, mx[0:1]))[0] for _ in range(3))
        # the part of the build after the event the statistics wait for (scan + fill)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        e1 = torch.cuda.Event(enable_timing=True)
        eng.ops.csr(state._table, n, k, s.lo, s.hi, mx[0:1], counted=ev)
        e1.record()
        torch.cuda.synchronize()
        tails.append(ev.elapsed_time(e1))
        csr = eng.ops.csr(state._table, n, k, s.lo, s.hi, mx[0:1])
        max_indeg = int(mx[0].item())
        out = torch.empty((s.hi - s.lo, k), dtype=torch.int32, device=dev)
        tally = torch.zeros(4, dtype=torch.int64, device=dev)
        bound = state._bound[1][s.lo:s.hi] if state._bound is not None else None
        bout = torch.empty(max(s.hi - s.lo, 1), dtype=torch.float32, device=dev)
        eng.ops.join(tabs, state._table, n, k, csr, max_indeg, out, tally, bound_in=bound, bound_out=bout)  # warm
        t_join = min(timed(lambda: eng.ops.join(tabs, state._table, n, k, csr, max_indeg, out, tally,
                                                bound_in=bound, bound_out=bout))[0] for _ in range(2))
        csr_ms.append(t_csr)
        join_ms.append(t_join)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    eng.ops.fcc(state._table, n, k, samples, cnt)
    t_fcc, _ = timed(lambda: eng.ops.fcc(state._table, n, k, samples, cnt))
    return max(csr_ms), max(join_ms), t_fcc, join_ms, min(tails)


st = b2.init_random_kout(b2.Dataset(pts), rs, cfg, b2.derive_rng(0, 2))
hist = []
per_p = {P: {"csr": 0.0, "join": 0.0, "fcc": 0.0, "sync": 0.0, "rounds": []} for P in P_LIST}
from paper_2202_00517_b200.descent import draw_fcc_schedule, _to_device  # noqa: E402

smp = _to_device(draw_fcc_schedule(n, k, cfg, cfg.resolved_max_rounds(n)), dev)
for r in range(1, cfg.resolved_max_rounds(n) + 1):
    for P in P_LIST:
        c, j, f, js, tail = shard_costs(st, P, smp[r - 1])
        acc = per_p[P]
        acc["csr"] += c
        acc["join"] += j
        acc["fcc"] += f
        acc["sync"] += (args.sync_us / 1e3 if P > 1 else 0.0) + max(0.0, args.host_us / 1e3 - tail)
        acc["rounds"].append({"round": r, "join_ms_per_rank": [round(x, 3) for x in js], "csr_ms": round(c, 3),
                              "csr_tail_ms": round(tail, 3)})
    st, s = b2.run_round(st, rs, cfg)
    hist.append(s)
    if len(hist) >= 2 and hist[-1].fcc <= hist[-2].fcc:
        break

base = None
for P in P_LIST:
    a = per_p[P]
    total = a["csr"] + a["join"] + a["fcc"] + a["sync"]
    base = base or total
    print(json.dumps({"ranks": P, "n": n, "d": d, "k": k, "rounds": len(hist),
                      "projected_ms": round(total, 3), "speedup_vs_1": round(base / total, 3),
                      "join_ms": round(a["join"], 3), "csr_ms": round(a["csr"], 3), "fcc_ms": round(a["fcc"], 3),
                      "sync_ms": round(a["sync"], 3), "per_round": a["rounds"]}), flush=True)
