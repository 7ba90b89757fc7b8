"""Device round engine: row shards, the per-round kernel sequence, and the
table exchange between ranks.

One process per GPU.  Rank r of P owns anchors [r*chunk, min((r+1)*chunk, n))
with chunk = ceil(n/P); every rank holds the full vector tables and the full
int32 friends table (padded to P*chunk rows so the NCCL all-gather is
in-place and equal-sized).  A round (run_round, descent.py:282-314) is:

  local join (own anchors -> own slice of the next table)     knnd_local_join
  exchange of the next table, all-reduce of the tallies        (P > 1, below)
  co-friend CSR of the next table for own targets              knnd_csr_build
  FCC count of the next table (replicated on every rank)       knnd_fcc
  one small device->host read: tallies, FCC count, max in-degree

The exchange (P > 1) is fused into the join by default: the next tables are a
ping-pong pair in symmetric memory (every rank maps every rank's copy over
NVLink), and the join kernel stores each finished row into every peer's copy
as it goes (knnd_local_join_peers) — the transfer overlaps the join, and a
device-side cross-rank barrier replaces the all-gather.  KNND_EXCHANGE=nccl
selects the plain in-place NCCL all-gather after the join instead.

The kernel calls go through an ``ops`` object; ``CudaOps`` is the product
(libknnd.so).  Tests inject a CPU stand-in to exercise the multi-rank logic
under the gloo backend without a GPU.
"""

from __future__ import annotations

import os
import sys
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    n: int

    @property
    def chunk(self) -> int:
        return -(-self.n // self.world)

    @property
    def lo(self) -> int:
        return min(self.rank * self.chunk, self.n)

    @property
    def hi(self) -> int:
        return min(self.lo + self.chunk, self.n)

    @property
    def padded_rows(self) -> int:
        return self.chunk * self.world


@dataclass
class Csr:
    indptr: torch.Tensor  # int64 (hi-lo+1,)
    indices: torch.Tensor  # int32 (n*K,)
    lo: int
    hi: int


# Workspace guard zones (KNND_GUARD=1; tests/test_checked.py): every workspace
# gets GUARD bytes of a known pattern on both sides, and check_guards() reports
# any that a kernel overwrote — the host-side half of the stand-in for
# compute-sanitizer (the device-side half is the checked build's bounds checks).
GUARD = 4096
_GUARD_BYTE = 0x5A
_guards: list = []


def workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    """A uint8 device workspace of at least nbytes (guarded under KNND_GUARD=1)."""
    nbytes = max(int(nbytes), 256)
    if os.environ.get("KNND_GUARD") != "1":
        return torch.empty(nbytes, dtype=torch.uint8, device=device)
    raw = torch.full((nbytes + 2 * GUARD,), _GUARD_BYTE, dtype=torch.uint8, device=device)
    _guards.append(raw)
    return raw[GUARD:GUARD + nbytes]


def check_guards() -> int:
    """Number of guard bytes overwritten since the workspaces were made (0 = clean)."""
    bad = 0
    for raw in _guards:
        n = raw.numel() - 2 * GUARD
        bad += int((raw[:GUARD] != _GUARD_BYTE).sum()) + int((raw[GUARD + n:] != _GUARD_BYTE).sum())
    return bad


class CudaOps:
    """The product kernel calls (libknnd.so) on one device's current stream."""

    def __init__(self, device: torch.device):
        self.device = device
        self._ws = {}
        self._side = None

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _side_stream(self) -> int:
        """The stream the join's big-table classes run on, concurrently with the
        rest (the library forks to it and joins back within the call)."""
        if self._side is None:
            self._side = torch.cuda.Stream(self.device)
        return self._side.cuda_stream

    def _workspace(self, key: str, nbytes: int) -> torch.Tensor:
        buf = self._ws.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = workspace(nbytes, self.device)
            self._ws[key] = buf
        return buf

    def csr(self, table: torch.Tensor, n: int, k: int, lo: int, hi: int, max_out: torch.Tensor | None,
            counted: "torch.cuda.Event | None" = None) -> Csr:
        """`counted` (optional) is recorded on the stream once max_out is final, before
        the scan and the fill of the build (knnd_csr_build_ev)."""
        indptr = torch.empty(hi - lo + 1, dtype=torch.int64, device=self.device)
        indices = torch.empty(max(n * k, 1), dtype=torch.int32, device=self.device)
        nbytes = _lib.load().knnd_csr_workspace_bytes(n, k, lo, hi)
        ws = self._workspace("csr", nbytes)
        _lib.call("knnd_csr_build_ev", table.data_ptr(), n, k, lo, hi, indptr.data_ptr(), indices.data_ptr(),
                  max_out.data_ptr() if max_out is not None else None, ws.data_ptr(), ws.numel(), self._stream(),
                  counted.cuda_event if counted is not None else None)
        return Csr(indptr, indices, lo, hi)

    def join(self, tabs, table: torch.Tensor, n: int, k: int, csr: Csr, max_indeg: int, out_rows: torch.Tensor,
             tally: torch.Tensor, out_kl: torch.Tensor | None = None, out_ucount: torch.Tensor | None = None,
             flags: int | None = None, bound_in: torch.Tensor | None = None,
             bound_out: torch.Tensor | None = None, peers=()) -> None:
        """knnd_local_join_peers (KL) / knnd_l2_local_join_peers (Euclidean), by
        the tables' metric; `peers` = device addresses of the other ranks'
        next tables (row 0), or empty."""
        if flags is None:
            flags = tabs.join_flags()
        nbytes = _lib.load().knnd_local_join_workspace_bytes(n, tabs.dplan, k, csr.lo, csr.hi, max_indeg)
        ws = self._workspace("join", nbytes)
        tabs.join(table, k, csr, max_indeg, out_rows, tally, out_kl, out_ucount, bound_in, bound_out, ws, flags,
                  self._stream(), peers=tuple(peers), side_stream=self._side_stream())

    def random_kout(self, state: tuple, n: int, k: int, table: torch.Tensor, out_meta: torch.Tensor,
                    bad: torch.Tensor) -> None:
        """numpy's PCG64 integers(0, n-1, (n, k)) + row shift on the device (knnd_random_kout).
        out_meta (int64, 2): [0] u32 values consumed, [1] number of rows with duplicates."""
        s, inc, has, uint = state
        m64 = (1 << 64) - 1
        nbytes = _lib.load().knnd_random_kout_workspace_bytes(n, k)
        ws = self._workspace("rng", nbytes)
        _lib.call("knnd_random_kout", s >> 64, s & m64, inc >> 64, inc & m64, has, uint, n, k, table.data_ptr(),
                  out_meta.data_ptr(), bad.data_ptr(), out_meta[1:].view(torch.int32).data_ptr(), ws.data_ptr(),
                  ws.numel(), self._stream())

    def fcc(self, table: torch.Tensor, n: int, k: int, samples: torch.Tensor, out_count: torch.Tensor) -> None:
        s = samples.shape[1]
        _lib.call("knnd_fcc", table.data_ptr(), n, k, samples[0].data_ptr(), samples[1].data_ptr(),
                  samples[2].data_ptr(), s, out_count.data_ptr(), self._stream())

    def sort_rows(self, tabs, rows: torch.Tensor, k: int, lo: int, hi: int, out_kl: torch.Tensor | None = None):
        # in place: each warp reads its row before writing it back
        tabs.sort_rows(rows, k, lo, hi, out_kl, self._stream())


class PeerTables:
    """The ping-pong pair of next tables of the fused exchange.

    bufs[i]   this rank's copy of table i, (padded_rows, K) int32
    peers[i]  the other ranks' copies of table i as this process addresses
              them (device pointers for CudaOps; tensors for the CPU stand-in)
    barrier(i) a cross-rank barrier on the current stream after which every
              copy of table i holds every rank's rows

    Round r reads one table and writes the other on every rank, so a copy is
    only overwritten after every rank has passed the barrier of the round that
    last read it.  A table returned in a KnnState stays valid until the round
    after next (descend_resident only hands out the final one)."""

    def __init__(self, bufs: list, peers: list, barrier: Callable[[int], None]):
        self.bufs, self.peers, self.barrier = bufs, peers, barrier
        # bumped whenever a round starts writing table i: a state holding an
        # older generation of table i has been overwritten (KnnState checks)
        self.gen = [0, 0]

    def pick(self, table: torch.Tensor) -> int:
        """Index of the table the round reading `table` writes."""
        return 1 if table.data_ptr() == self.bufs[0].data_ptr() else 0

    def index_of(self, table: torch.Tensor) -> int | None:
        """i if `table` is (a view starting at) this rank's copy of table i."""
        for i, b in enumerate(self.bufs):
            if table.data_ptr() == b.data_ptr():
                return i
        return None

    def begin_write(self, i: int) -> None:
        self.gen[i] += 1


_PEER_CACHE: dict = {}


def symmetric_peer_tables(eng: "Engine") -> PeerTables:
    """Both tables in torch symmetric memory (CUDA IPC mappings of every rank's
    buffer over NVLink).  The mapping is a collective (a rendezvous of every
    rank), so it is made once per (device, table shape, group) and reused by
    later descents: descend_resident hands out its final table as a private
    copy, and an intermediate state (on_round) raises once a later round has
    reused its table (PeerTables.gen)."""
    import torch.distributed._symmetric_memory as symm

    group = eng.group if eng.group is not None else dist.group.WORLD
    key = (eng.device, eng.shard.padded_rows, eng.k, group.group_name, id(group))
    if key in _PEER_CACHE:
        return _PEER_CACHE[key]
    bufs, handles = [], []
    for _ in range(2):
        t = symm.empty((eng.shard.padded_rows, eng.k), dtype=torch.int32, device=eng.device)
        handles.append(symm.rendezvous(t, group))
        bufs.append(t)
    me, world = eng.shard.rank, eng.shard.world
    peers = [[int(h.buffer_ptrs[r]) for r in range(world) if r != me] for h in handles]
    pt = PeerTables(bufs, peers, lambda i: handles[i].barrier(channel=0))
    _PEER_CACHE[key] = pt
    return pt


def peer_capable(eng: "Engine") -> bool:
    """This rank can map every other rank's device memory: torch symmetric
    memory is importable and CUDA peer access to each rank's device exists
    (device indices gathered over the group)."""
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
    except Exception:
        ok = False
    else:
        ok = eng.device.type == "cuda"
    idx = torch.tensor([eng.device.index if eng.device.index is not None else -1], dtype=torch.int64,
                       device=eng.device)
    allidx = [torch.empty_like(idx) for _ in range(eng.shard.world)]
    dist.all_gather(allidx, idx, group=eng.group)
    if ok:
        me = eng.device.index
        for t in allidx:
            other = int(t.item())
            if other != me and (other < 0 or not torch.cuda.can_device_access_peer(me, other)):
                ok = False
    return ok


def exchange_mode(eng: "Engine") -> str:
    """'peer' (fused stores, default for P > 1 on CUDA + NCCL) or 'nccl'."""
    want = os.environ.get("KNND_EXCHANGE", "peer")
    if want not in ("peer", "nccl"):
        raise ValueError(f"KNND_EXCHANGE must be 'peer' or 'nccl', got {want!r}")
    if eng.shard.world == 1 or eng.device.type != "cuda" or dist.get_backend(eng.group) != "nccl":
        return "nccl"
    return want


@dataclass
class RoundResult:
    csr: Csr
    comparisons: int
    changed: int
    bad: int
    fcc_count: int
    max_indeg: int
    bound: torch.Tensor | None = None  # per own row: largest screened value of the new row


class Engine:
    """Shard-aware round engine for one device (and one rank)."""

    def __init__(self, n: int, k: int, device: torch.device, group=None, ops=None):
        self.n, self.k = n, k
        self.device = device
        self.group = group
        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            rank, world = 0, 1
        self.shard = Shard(rank, world, n)
        self.ops = ops if ops is not None else CudaOps(device)
        # int64 slots: [0:4] tally (comparisons, changed, bad, -), [4] = int32 (fcc count, max in-degree),
        # [5] this rank's comparisons
        self.stats = torch.zeros(8, dtype=torch.int64, device=device)
        self._stats32 = self.stats.view(torch.int32)
        # The round's statistics are read behind an event recorded inside the CSR build, as soon
        # as the max in-degree is final: the host decides (stop test, next plan) and queues the
        # next round while the build's scan and fill — two thirds of it — still run, so the
        # device does not idle for the host's latency each round (CUDA ops only).
        self._stats_ev = self._stats_stream = self._stats_host = None
        if isinstance(self.ops, CudaOps):
            self._stats_stream = torch.cuda.Stream(device)
            self._stats_ev = torch.cuda.Event()
            self._stats_ev.record(torch.cuda.current_stream(device))  # (creates the CUDA event: its handle is passed on)
            self._stats_host = torch.zeros(8, dtype=torch.int64).pin_memory()
        # optional CUDA-event bracketing of each local join (bench.py roofline)
        self.join_events: list | None = None
        self.peer: PeerTables | None = None  # fused exchange (P > 1), see enable_peer_exchange

    def enable_peer_exchange(self, peer: PeerTables | None = None) -> bool:
        """Switch rounds to the fused exchange (idempotent).  Without an explicit
        `peer`, maps symmetric-memory tables when exchange_mode() says so; if
        that mapping fails the engine keeps the NCCL all-gather and says why."""
        if peer is not None:
            self.peer = peer
        elif self.peer is None and exchange_mode(self) == "peer":
            # agree on capability before the rendezvous (a collective every rank
            # must enter), so no rank waits in it for one that will not come
            can = torch.tensor([int(peer_capable(self))], dtype=torch.int32, device=self.device)
            dist.all_reduce(can, op=dist.ReduceOp.MIN, group=self.group)
            if int(can.item()) == 0:
                print("knnd: a rank cannot map its peers' tables; using the NCCL all-gather", file=sys.stderr)
                return False
            try:
                self.peer = symmetric_peer_tables(self)
            except Exception as exc:  # e.g. no P2P / IPC between these devices
                print(f"knnd: fused peer exchange unavailable ({type(exc).__name__}: {exc}); "
                      "using the NCCL all-gather", file=sys.stderr)
            # every rank must take the same exchange, or the rounds deadlock
            ok = torch.tensor([int(self.peer is not None)], dtype=torch.int32, device=self.device)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
            if int(ok.item()) == 0 and self.peer is not None:
                print("knnd: another rank could not map the peer tables; using the NCCL all-gather",
                      file=sys.stderr)
                self.peer = None
        return self.peer is not None

    # -- tables -----------------------------------------------------------
    def alloc_table(self) -> torch.Tensor:
        return torch.empty((self.shard.padded_rows, self.k), dtype=torch.int32, device=self.device)

    def own_rows(self, table: torch.Tensor) -> torch.Tensor:
        s = self.shard
        return table[s.lo:s.hi]

    def exchange(self, table: torch.Tensor) -> None:
        """In-place all-gather of every rank's slice (NCCL over NVLink)."""
        s = self.shard
        if s.world == 1:
            return
        flat = table.view(-1)
        mine = flat[s.rank * s.chunk * self.k:(s.rank + 1) * s.chunk * self.k]
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(flat, mine, group=self.group)  # in place
        elif flat.is_cuda:  # gloo (tests: several ranks on one device): through host memory
            host = flat.cpu()
            dist.all_gather_into_tensor(host, host[s.rank * s.chunk * self.k:(s.rank + 1) * s.chunk * self.k].clone(),
                                        group=self.group)
            flat.copy_(host)
        else:
            dist.all_gather_into_tensor(flat, mine.clone(), group=self.group)

    def all_reduce(self, t: torch.Tensor) -> None:
        """Sum over ranks (NCCL; gloo stages CUDA tensors through host memory)."""
        if dist.get_backend(self.group) != "nccl" and t.is_cuda:
            host = t.cpu()
            dist.all_reduce(host, group=self.group)
            t.copy_(host)
        else:
            dist.all_reduce(t, group=self.group)

    def upload_rows(self, host_rows: np.ndarray, table: torch.Tensor) -> int:
        """Copy this rank's rows of a host (n, K) table into `table`; returns bytes copied."""
        s = self.shard
        src = torch.from_numpy(np.ascontiguousarray(host_rows[s.lo:s.hi], dtype=np.int32))
        if self.device.type == "cuda":
            src = src.pin_memory()
        self.own_rows(table).copy_(src, non_blocking=True)
        return src.numel() * 4

    def upload_table(self, host: np.ndarray) -> torch.Tensor:
        """A full host table onto the device (every rank uploads all rows)."""
        t = self.alloc_table()
        src = torch.from_numpy(np.ascontiguousarray(host, dtype=np.int32))
        if self.device.type == "cuda":
            src = src.pin_memory()
        t[: self.n].copy_(src, non_blocking=True)
        return t

    # -- kernels ----------------------------------------------------------
    def build_csr(self, table: torch.Tensor) -> tuple[Csr, int]:
        s = self.shard
        mx = self._stats32[9:10]
        csr = self.ops.csr(table, self.n, self.k, s.lo, s.hi, mx)
        return csr, int(mx.item())

    def init_rows(self, tabs, draws: np.ndarray) -> torch.Tensor:
        """_sort_rows_by_anchor (descent.py:163-174) for own rows, then exchange."""
        s = self.shard
        table = self.alloc_table()
        self.upload_rows(draws, table)
        self.ops.sort_rows(tabs, self.own_rows(table), self.k, s.lo, s.hi)
        self.exchange(table)
        return table

    def round(self, tabs, table: torch.Tensor, csr: Csr, max_indeg: int, samples: torch.Tensor | None,
              out_kl: torch.Tensor | None = None, out_ucount: torch.Tensor | None = None,
              bound: torch.Tensor | None = None) -> tuple[torch.Tensor, RoundResult]:
        """One round.  `bound` is the RoundResult.bound of the round that produced
        `table` with the same `tabs` (or None); the new one is returned."""
        tally = self.stats[0:4]
        tally.zero_()
        if self.peer is not None:
            ip = self.peer.pick(table)
            nxt, peers = self.peer.bufs[ip], self.peer.peers[ip]
            self.peer.begin_write(ip)
        else:
            nxt, peers = self.alloc_table(), ()
        s = self.shard
        bound_out = torch.empty(max(s.hi - s.lo, 1), dtype=torch.float32, device=self.device)
        ev = None
        if self.join_events is not None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        self.ops.join(tabs, table, self.n, self.k, csr, max_indeg, self.own_rows(nxt), tally, out_kl, out_ucount,
                      bound_in=bound, bound_out=bound_out, peers=peers)
        if ev is not None:
            ev[1].record()
        self.stats[5:6].copy_(tally[0:1])  # this rank's comparisons (before the all-reduce)
        if self.shard.world > 1:
            if self.peer is not None:
                self.peer.barrier(ip)  # every rank's rows are in every copy
            else:
                self.exchange(nxt)
            self.all_reduce(tally)
        if samples is not None:
            self.ops.fcc(nxt, self.n, self.k, samples, self._stats32[8:9])
        if self._stats_ev is not None:
            csr_next = self.ops.csr(nxt, self.n, self.k, s.lo, s.hi, self._stats32[9:10], counted=self._stats_ev)
            self._stats_stream.wait_event(self._stats_ev)
            with torch.cuda.stream(self._stats_stream):
                self._stats_host.copy_(self.stats, non_blocking=True)
            self._stats_stream.synchronize()  # the one synchronisation of the round
            host = self._stats_host.clone()
        else:
            csr_next = self.ops.csr(nxt, self.n, self.k, s.lo, s.hi, self._stats32[9:10])
            host = self.stats.cpu()  # the one synchronisation of the round
        h32 = host.view(torch.int32)
        if ev is not None:
            self.join_events.append((ev[0].elapsed_time(ev[1]), int(host[5])))
        return nxt, RoundResult(csr_next, int(host[0]), int(host[1]), int(host[2]), int(h32[8]), int(h32[9]),
                                bound_out)

    def fcc(self, table: torch.Tensor, samples: torch.Tensor) -> int:
        self.ops.fcc(table, self.n, self.k, samples, self._stats32[8:9])
        return int(self._stats32[8].item())
