"""K-NN descent on B200 — the drop-in for rankdescent.descent (descent.py:1-391).

Same entry points, arguments, return types and errors as the reference:

  run(dataset, rs, cfg)          -> (friends int64 (n,K) read-only, [RoundStats])
  run_to_fixed_point(...)        -> same, stops when no row changes
  run_round(state, rs, cfg)      -> (KnnState, RoundStats)
  init_random_kout(ds, rs, cfg, rng) -> KnnState
  friend_clustering_rate(state, S, rng) -> float
  propose_new_friend_set(x, state, rs)  -> the new row of x

Every random draw is made on the host with the reference's own numpy
substreams (derive_rng, descent.py:43-45), so inputs and samples are bitwise
those of the reference; all per-round arithmetic runs in the sm_100a kernels
of libknnd.so.  The friends table and its co-friend CSR stay resident in HBM
between rounds; ``KnnState.friends`` downloads lazily.

Under ``torchrun`` (torch.distributed initialised) every rank calls the same
function; anchors are row-sharded and the table is all-gathered each round
(see engine.py).  Results do not depend on the rank count.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from .core import ConfigError, Dataset, ItemId
from .engine import Csr, Engine
from .similarity import device_for, device_tables_for

_SEED_MASK = 0xFFFFFFFFFFFFFFFF

STREAM_DATA = 1
STREAM_INIT = 2
STREAM_FCC = 3
STREAM_RECALL = 4
STREAM_WITNESS = 5

MAX_K = 64  # the device join's limit (one or two 32-lane selection registers per lane)


def derive_rng(seed: int, *path: int) -> np.random.Generator:
    """descent.py:43-45 — the per-purpose numpy substream."""
    return np.random.default_rng(np.random.SeedSequence([seed & _SEED_MASK, *path]))


def round_budget(n: int, k: int) -> int:
    """descent.py:48-57 — 2 * ceil(log_k n) with the float guard."""
    if n < 2 or k < 2:
        raise ConfigError(f"round budget needs n >= 2 and k >= 2, got n={n}, k={k}")
    return 2 * math.ceil(math.log(n) / math.log(k) - 1e-9)


@dataclass
class DescentConfig:
    """descent.py:60-97.  worker_count is accepted for compatibility; on the
    device it never changes results (nor, here, the schedule)."""

    k: int
    fcc_sample_count: int = 1000
    max_rounds: int | None = None
    seed: int = 0
    worker_count: int | str = 1

    def __post_init__(self) -> None:
        if self.k < 2:
            raise ConfigError(f"k must be >= 2 (the stopping sampler draws friend pairs), got {self.k}")
        if self.k > MAX_K:  # a device limit the reference does not have: refuse before any upload
            raise ConfigError(f"k must be <= {MAX_K} on the B200 engine, got {self.k}")
        if self.fcc_sample_count < 1:
            raise ConfigError(f"fcc_sample_count must be >= 1, got {self.fcc_sample_count}")
        if self.max_rounds is not None and self.max_rounds < 1:
            raise ConfigError(f"max_rounds must be >= 1, got {self.max_rounds}")
        if isinstance(self.worker_count, str):
            if self.worker_count != "auto":
                raise ConfigError(f'worker_count must be a positive int or "auto", got {self.worker_count!r}')
        elif self.worker_count < 1:
            raise ConfigError(f"worker_count must be >= 1, got {self.worker_count}")

    def resolved_max_rounds(self, n: int) -> int:
        return self.max_rounds if self.max_rounds is not None else round_budget(n, self.k) + 4

    def resolved_workers(self) -> int:
        return (os.cpu_count() or 1) if self.worker_count == "auto" else int(self.worker_count)


@dataclass
class RoundStats:
    """descent.py:100-108."""

    round_index: int
    wall_clock_sec: float
    fcc: float
    comparisons: int
    changed_friend_sets: int


def _device(device=None) -> torch.device:
    if device is not None:
        dev = torch.device(device)
    else:
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 descent engine has no CPU fallback")
        dev = torch.device("cuda", torch.cuda.current_device())
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


class KnnState:
    """Device-resident snapshot of the friends digraph plus its co-friend CSR
    (descent.py:111-148).  Constructing one from a host array uploads it and
    builds the CSR on the GPU; rounds produce new states without host copies.
    """

    def __init__(self, friends, round_index: int = 0, fcc_history: Sequence[float] = (), *, device=None):
        arr = np.array(friends, dtype=np.int64)
        if arr.ndim != 2:
            raise ValueError(f"friends must be an (n, K) array, got shape {arr.shape}")
        n, k = arr.shape
        if arr.size and (arr.min() < 0 or arr.max() >= n):
            raise ValueError("friends ids must lie in [0, n)")
        arr.flags.writeable = False
        eng = Engine(n, k, _device(device))
        table = eng.upload_table(arr)
        csr, mx = eng.build_csr(table)
        self._bind(eng, table, csr, mx, round_index, tuple(fcc_history))
        self._host = arr

    @classmethod
    def _from_device(cls, eng: Engine, table, csr: Csr, max_indeg: int, round_index: int, hist,
                     bound=None) -> "KnnState":
        st = cls.__new__(cls)
        st._bind(eng, table, csr, max_indeg, round_index, tuple(hist))
        st._bound = bound
        if eng.peer is not None:  # a ping-pong table of the fused exchange: remember its generation
            i = eng.peer.index_of(table)
            if i is not None:
                st._peer_ref = (eng.peer, i, eng.peer.gen[i])
        return st

    def _bind(self, eng, table, csr, max_indeg, round_index, hist):
        self._engine = eng
        self._table_t = table
        self._peer_ref = None
        self._csr = csr
        self._max_indeg = max_indeg
        self.round = round_index
        self.fcc_history = hist
        self._host = None
        self._host_csr = None
        # (tables, per-row bound) from the round that produced this table; a
        # hint for the next join with the same tables, never shared or mutated
        self._bound = None

    @property
    def _table(self) -> torch.Tensor:
        """The device table; raises if the fused exchange has since reused it
        (the reference's KnnState is immutable: never hand out another table)."""
        ref = self._peer_ref
        if ref is not None and ref[0].gen[ref[1]] != ref[2]:
            raise RuntimeError(f"the device table of this round-{self.round} KnnState was reused by a later round "
                               "of the fused exchange; read .friends before the round after next")
        return self._table_t

    def _detach(self) -> None:
        """Move the table into a private device copy (off the ping-pong pair)."""
        if self._peer_ref is not None:
            self._table_t = self._table.clone()
            self._peer_ref = None

    # -- reference attributes ----------------------------------------------
    @property
    def n(self) -> int:
        return self._engine.n

    @property
    def k(self) -> int:
        return self._engine.k

    @property
    def device(self) -> torch.device:
        return self._engine.device

    @property
    def friends(self) -> np.ndarray:
        if self._host is None:  # widen on the device, one D2H copy into (cached) pinned memory
            dev64 = self._table[: self.n].to(torch.int64)
            if dev64.is_cuda:
                pinned = torch.empty(dev64.shape, dtype=torch.int64, pin_memory=True)
                pinned.copy_(dev64)
                host = pinned.numpy()
            else:
                host = dev64.numpy().copy()
            host.flags.writeable = False
            self._host = host
        return self._host

    def _cofriend_csr(self):
        if self._host_csr is None:
            s = self._engine.shard
            if s.world != 1:
                raise RuntimeError("the host CSR view is only available for single-rank states")
            ptr = self._csr.indptr.cpu().numpy().astype(np.int64)
            idx = self._csr.indices[: ptr[-1]].cpu().numpy().astype(np.int64)
            for t in range(self.n):  # the device leaves segment order unspecified; present it ascending
                seg = idx[ptr[t]:ptr[t + 1]]
                seg.sort()
            self._host_csr = (ptr, idx)
        return self._host_csr

    @property
    def cof_indptr(self) -> np.ndarray:
        return self._cofriend_csr()[0]

    @property
    def cof_indices(self) -> np.ndarray:
        return self._cofriend_csr()[1]

    def friends_of(self, x: ItemId) -> np.ndarray:
        return self.friends[x]

    def cofriends_of(self, x: ItemId) -> np.ndarray:
        ptr, idx = self._cofriend_csr()
        return idx[ptr[x]:ptr[x + 1]]

    def friends_dict(self) -> dict[int, set[int]]:
        return {x: set(map(int, row)) for x, row in enumerate(self.friends)}

    def cofriends_dict(self) -> dict[int, set[int]]:
        return {x: set(map(int, self.cofriends_of(x))) for x in range(self.n)}


# ---------------------------------------------------------------------------
# host-side draws (the reference's RNG consumption, bit for bit)


def random_kout_draws(n: int, k: int, rng: np.random.Generator) -> np.ndarray:
    """descent.py:193-212 — K distinct uniform non-self targets per row.

    Rejection rows are re-checked only after a redraw (rows without duplicates
    never change), which consumes the stream exactly as the reference does."""
    anchors = np.arange(n, dtype=np.int64)[:, None]
    if n - 1 > 2 * k * k:
        draws = rng.integers(0, n - 1, size=(n, k), dtype=np.int64)
        draws += draws >= anchors
        srt = np.sort(draws, axis=1)
        bad = np.nonzero((srt[:, 1:] == srt[:, :-1]).any(axis=1))[0]
        while bad.size:
            redraw = rng.integers(0, n - 1, size=(bad.size, k), dtype=np.int64)
            redraw += redraw >= bad[:, None]
            draws[bad] = redraw
            srt = np.sort(redraw, axis=1)
            bad = bad[(srt[:, 1:] == srt[:, :-1]).any(axis=1)]
        return draws
    draws = np.empty((n, k), dtype=np.int64)
    for x in range(n):
        row = rng.permutation(n - 1)[:k]
        row += row >= x
        draws[x] = row
    return draws


_M64 = (1 << 64) - 1
_M128 = (1 << 128) - 1
_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645  # PCG64 (XSL-RR 128/64) multiplier


def _pcg_output(s: int) -> int:
    x = (s >> 64) ^ (s & _M64)
    rot = s >> 122
    return ((x >> rot) | (x << ((64 - rot) & 63))) & _M64


def _pcg_advance(s: int, inc: int, steps: int) -> int:
    """The PCG64 state after `steps` 64-bit outputs (LCG jump-ahead)."""
    a, c = _PCG_MULT, inc
    acc_a, acc_c = 1, 0
    while steps:
        if steps & 1:
            acc_a, acc_c = (a * acc_a) & _M128, (a * acc_c + c) & _M128
        c = (a * c + c) & _M128
        a = (a * a) & _M128
        steps >>= 1
    return (acc_a * s + acc_c) & _M128


def device_random_kout(eng: Engine, n: int, k: int, rng: np.random.Generator, table: torch.Tensor) -> bool:
    """descent.py:194-205 with the first (n, K) draw made on the device by a
    bit-exact replica of numpy's PCG64 + Lemire stream (knnd_random_kout); the
    numpy generator is then advanced past the values the device consumed and
    the rejection redraws of rows with duplicates run on the host, exactly as
    the reference does them.  Returns False (nothing done) when the generator is
    not PCG64 or the ops have no device path."""
    finish = device_random_kout_async(eng, n, k, rng, table)
    return finish is not None and finish()


def device_random_kout_async(eng: Engine, n: int, k: int, rng: np.random.Generator, table: torch.Tensor):
    """device_random_kout split at its one synchronisation: launches the draw
    kernel and returns a `finish()` that completes the generator bookkeeping
    and the duplicate-row redraws (returns True), or None when there is no
    device path.  `rng` must not be used in between."""
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64" or not hasattr(eng.ops, "random_kout") or n - 1 > 0xFFFFFFFF:
        return None
    s0, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    has, uint = int(st["has_uint32"]), int(st["uinteger"])
    meta = torch.zeros(2, dtype=torch.int64, device=eng.device)
    bad_dev = torch.empty(n, dtype=torch.int32, device=eng.device)
    eng.ops.random_kout((s0, inc, has, uint), n, k, table, meta, bad_dev)
    return lambda: _finish_random_kout(eng, n, k, rng, table, meta, bad_dev, s0, inc, has)


def _finish_random_kout(eng, n, k, rng, table, meta, bad_dev, s0, inc, has) -> bool:
    consumed, nbad = (int(v) for v in meta.cpu().tolist())  # nbad: an int32 in the low half of meta[1]
    fresh = consumed - has
    if has and fresh < 0:
        fresh = 0
    s1 = _pcg_advance(s0, inc, (fresh + 1) // 2)
    left = fresh % 2 == 1
    rng.bit_generator.state = {"bit_generator": "PCG64", "state": {"state": s1, "inc": inc},
                               "has_uint32": 1 if left else 0, "uinteger": (_pcg_output(s1) >> 32) if left else 0}
    if nbad:
        bad = np.sort(bad_dev[:nbad].cpu().numpy().astype(np.int64))
        rows = bad.copy()
        fixed = {}
        while bad.size:  # descent.py:198-205, restricted to the rows that can still change
            redraw = rng.integers(0, n - 1, size=(bad.size, k), dtype=np.int64)
            redraw += redraw >= bad[:, None]
            for r, row in zip(bad, redraw):
                fixed[int(r)] = row
            srt = np.sort(redraw, axis=1)
            bad = bad[(srt[:, 1:] == srt[:, :-1]).any(axis=1)]
        vals = torch.from_numpy(np.stack([fixed[int(r)] for r in rows]).astype(np.int32)).to(eng.device)
        table[torch.from_numpy(rows).to(eng.device)] = vals
    return True


def fcc_samples(n: int, k: int, count: int, rng: np.random.Generator) -> np.ndarray:
    """descent.py:330-333 — (3, count) int32: anchors, slot i, slot j != i."""
    xs = rng.integers(0, n, size=count)
    i = rng.integers(0, k, size=count)
    j = rng.integers(0, k - 1, size=count)
    j += j >= i
    return np.stack([xs, i, j]).astype(np.int32)


def _to_device(a: np.ndarray, device: torch.device) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a))
    if device.type == "cuda":
        t = t.pin_memory()
    return t.to(device, non_blocking=True)


# ---------------------------------------------------------------------------
# the reference entry points


def init_random_kout(dataset: Dataset, rs, cfg: DescentConfig, rng: np.random.Generator, device=None) -> KnnState:
    """descent.py:177-213 — random K-out digraph, rows ordered by (score, draw position)."""
    n = len(dataset)
    k = cfg.k
    if n <= k:
        raise ConfigError(f"need n > k, got n={n}, k={k}")
    tabs = device_tables_for(rs, device)
    eng = Engine(n, k, tabs.device)
    table = eng.alloc_table()
    if not (n - 1 > 2 * k * k and device_random_kout(eng, n, k, rng, table)):
        eng.upload_rows(random_kout_draws(n, k, rng), table)
    s = eng.shard
    eng.ops.sort_rows(tabs, eng.own_rows(table), k, s.lo, s.hi)
    eng.exchange(table)
    csr, mx = eng.build_csr(table)
    return KnnState._from_device(eng, table, csr, mx, 0, ())


def _check_state(state: KnnState) -> None:
    if not isinstance(state, KnnState):
        raise TypeError(f"expected a paper_2202_00517_b200 KnnState, got {type(state).__name__}")


def _round(state: KnnState, tabs, samples_dev, sample_count: int, round_index: int):
    eng = state._engine
    bound = state._bound[1] if state._bound is not None and state._bound[0] is tabs else None
    nxt, res = eng.round(tabs, state._table, state._csr, state._max_indeg, samples_dev, bound=bound)
    if res.bad:
        raise RuntimeError(f"local join saw {res.bad} anchors with fewer than K candidates (malformed table)")
    rate = res.fcc_count / sample_count
    new_state = KnnState._from_device(eng, nxt, res.csr, res.max_indeg, round_index, state.fcc_history + (rate,),
                                      (tabs, res.bound))
    return new_state, res, rate


def run_round(state: KnnState, rs, cfg: DescentConfig) -> tuple[KnnState, RoundStats]:
    """descent.py:282-314 — one synchronous round against the snapshot."""
    _check_state(state)
    t0 = time.perf_counter()
    tabs = device_tables_for(rs, state.device)
    r = state.round + 1
    smp = fcc_samples(state.n, state.k, cfg.fcc_sample_count, derive_rng(cfg.seed, STREAM_FCC, r))
    new_state, res, rate = _round(state, tabs, _to_device(smp, state.device), cfg.fcc_sample_count, r)
    stats = RoundStats(r, time.perf_counter() - t0, rate, res.comparisons, res.changed)
    return new_state, stats


def friend_clustering_rate(state: KnnState, sample_count: int, rng: np.random.Generator) -> float:
    """descent.py:317-338 — sampled friend clustering rate, counted on the GPU."""
    _check_state(state)
    if state.k < 2:
        raise ConfigError(f"friend clustering rate needs k >= 2, got {state.k}")
    if sample_count < 1:
        raise ConfigError(f"sample_count must be >= 1, got {sample_count}")
    smp = fcc_samples(state.n, state.k, sample_count, rng)
    cnt = state._engine.fcc(state._table, _to_device(smp, state.device))
    return cnt / sample_count


def candidate_set(x: ItemId, state: KnnState) -> np.ndarray:
    """descent.py:216-227 — x's new acquaintances: cofriends, friends of friends
    and friends of cofriends, unique and sorted by id, without x and without
    x's current friends (the comparator engine's candidate set; the device
    join ranks the superset that keeps the friends, descent.py:230-242)."""
    _check_state(state)
    friends = state.friends
    frs = friends[x]
    cof = state.cofriends_of(x)
    cand = np.unique(np.concatenate((cof, friends[frs].ravel(), friends[cof].ravel())))
    mask = cand != x
    mask &= ~np.isin(cand, frs)
    return cand[mask]


def propose_new_friend_set(x: ItemId, state: KnnState, rs) -> np.ndarray:
    """descent.py:252-259 — the K best of x's friends and candidates, best first."""
    _check_state(state)
    eng = state._engine
    s = eng.shard
    if not (s.lo <= x < s.hi):
        raise ValueError(f"anchor {x} is not owned by this rank")
    tabs = device_tables_for(rs, state.device)
    sub = Csr(state._csr.indptr[x - s.lo:], state._csr.indices, x, x + 1)
    out = torch.empty((1, state.k), dtype=torch.int32, device=state.device)
    tally = torch.zeros(4, dtype=torch.int64, device=state.device)
    eng.ops.join(tabs, state._table, state.n, state.k, sub, state._max_indeg, out, tally)
    return out[0].cpu().numpy().astype(np.int64)


def draw_fcc_schedule(n: int, k: int, cfg: DescentConfig, max_rounds: int, first: int = 1) -> np.ndarray:
    """Every round's FCC sample is a function of (seed, round) only
    (descent.py:305): the samples of rounds first..max_rounds, (R, 3, S) int32."""
    return np.stack([fcc_samples(n, k, cfg.fcc_sample_count, derive_rng(cfg.seed, STREAM_FCC, r))
                     for r in range(first, max_rounds + 1)])


class FccSchedule:
    """The device copies of the rounds' FCC samples, drawn CHUNK rounds at a
    time when a round first asks for them: the cost follows the rounds actually
    run, not the round cap (run_to_fixed_point's cap can be large).
    ``sched[r - 1]`` is round r's (3, S) int32 sample on the device."""

    CHUNK = 4

    def __init__(self, n: int, k: int, cfg: DescentConfig, max_rounds: int, device: torch.device):
        self.n, self.k, self.cfg, self.max_rounds, self.device = n, k, cfg, max_rounds, device
        self._chunks: dict[int, torch.Tensor] = {}

    def __len__(self) -> int:
        return self.max_rounds

    def __getitem__(self, i: int) -> torch.Tensor:
        if not 0 <= i < self.max_rounds:
            raise IndexError(f"round {i + 1} is past the schedule's {self.max_rounds} rounds")
        c = i // self.CHUNK
        dev = self._chunks.get(c)
        if dev is None:
            first = c * self.CHUNK + 1
            last = min(first + self.CHUNK - 1, self.max_rounds)
            dev = _to_device(draw_fcc_schedule(self.n, self.k, self.cfg, last, first), self.device)
            self._chunks = {c: dev}  # earlier chunks are done with
        return dev[i - c * self.CHUNK]


def descend_resident(eng: Engine, tabs, table: torch.Tensor, samples_dev: torch.Tensor, sample_count: int,
                     max_rounds: int, stop_on_fixed_point: bool = False, on_round=None):
    """The round loop of _run_rounds (descent.py:341-362) over device-resident
    inputs: `table` holds the unsorted initial draws (own rows at least).
    Sorts the initial rows (K6), then runs rounds until the FCC stalls (or no
    row changes).  Returns (final KnnState, [RoundStats])."""
    s = eng.shard
    if s.world > 1:
        eng.enable_peer_exchange()  # fused join + table exchange when the ranks can map each other
    eng.ops.sort_rows(tabs, eng.own_rows(table), eng.k, s.lo, s.hi)
    eng.exchange(table)
    csr, mx = eng.build_csr(table)
    state = KnnState._from_device(eng, table, csr, mx, 0, ())
    history: list[RoundStats] = []
    for r in range(1, max_rounds + 1):
        t0 = time.perf_counter()
        state, res, rate = _round(state, tabs, samples_dev[r - 1], sample_count, r)
        history.append(RoundStats(r, time.perf_counter() - t0, rate, res.comparisons, res.changed))
        if on_round is not None:
            on_round(state, history[-1])
        if stop_on_fixed_point:
            if res.changed == 0:
                break
        elif len(history) >= 2 and history[-1].fcc <= history[-2].fcc:
            break
    state._detach()  # the ping-pong tables are reused by the next descent
    return state, history


def _run_rounds(dataset: Dataset, rs, cfg: DescentConfig, max_rounds: int, stop_on_fixed_point: bool):
    n = len(dataset)
    k = cfg.k
    if n <= k:
        raise ConfigError(f"need n > k, got n={n}, k={k}")
    # the device draws, the host FCC schedule and the table upload overlap: the
    # draw kernel runs while the host draws the schedule and stages the points
    eng = Engine(n, k, device_for(rs))
    table = eng.alloc_table()
    rng = derive_rng(cfg.seed, STREAM_INIT)
    finish = device_random_kout_async(eng, n, k, rng, table) if n - 1 > 2 * k * k else None
    smp_dev = FccSchedule(n, k, cfg, max_rounds, eng.device)
    smp_dev[0]  # the first rounds' samples are drawn while the draw kernel runs
    tabs = device_tables_for(rs, eng.device)
    if not (finish is not None and finish()):
        eng.upload_rows(random_kout_draws(n, k, rng), table)
    state, history = descend_resident(eng, tabs, table, smp_dev, cfg.fcc_sample_count, max_rounds,
                                      stop_on_fixed_point)
    return state.friends, history


def run(dataset: Dataset, rs, cfg: DescentConfig) -> tuple[np.ndarray, list[RoundStats]]:
    """descent.py:365-373 — init, then rounds until the clustering rate stalls."""
    return _run_rounds(dataset, rs, cfg, cfg.resolved_max_rounds(len(dataset)), stop_on_fixed_point=False)


def run_to_fixed_point(dataset: Dataset, rs, cfg: DescentConfig) -> tuple[np.ndarray, list[RoundStats]]:
    """descent.py:376-391 — rounds until no row changes (cap 8*budget+16)."""
    cap = cfg.max_rounds if cfg.max_rounds is not None else 8 * round_budget(len(dataset), cfg.k) + 16
    return _run_rounds(dataset, rs, cfg, cap, stop_on_fixed_point=True)
