"""numpy restatement of the reference's hot path (TEST INFRASTRUCTURE ONLY).

Each function states which reference function it restates
(paths relative to /root/reference/pkg/src/rankdescent/).  The restatement is
deliberately literal in *semantics* — same RNG streams, same np.unique /
stable-argsort ordering, same einsum scoring — so its outputs are bitwise
equal to the reference's; tests/test_oracle.py pins that against the golden
fixtures recorded from the reference itself.
"""

from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
TAG_DATA, TAG_INIT, TAG_FCC, TAG_RECALL = 1, 2, 3, 4


# --------------------------------------------------------------------------
# RNG substreams and budget — descent.py:43-57


def substream(seed: int, *tags: int) -> np.random.Generator:
    """descent.py:43-45 derive_rng: Generator(PCG64(SeedSequence([seed mod 2^64, *tags])))."""
    return np.random.default_rng(np.random.SeedSequence([seed & MASK64, *tags]))


def budget(n: int, k: int) -> int:
    """descent.py:48-57 round_budget: 2 * ceil(log_k n), with the 1e-9 guard."""
    if n < 2 or k < 2:
        raise ValueError("budget needs n >= 2 and k >= 2")
    return 2 * math.ceil(math.log(n) / math.log(k) - 1e-9)


def round_cap(n: int, k: int, max_rounds: int | None = None) -> int:
    """descent.py:89-92 resolved_max_rounds."""
    return max_rounds if max_rounds is not None else budget(n, k) + 4


# --------------------------------------------------------------------------
# data and scoring — similarity.py:50-106, bench.py:125-127


def simplex_points(d: int, n: int, rng: np.random.Generator) -> np.ndarray:
    """similarity.py:50-77 with concentration 1: normalized unit exponentials,
    zero draws replaced by fresh exponentials."""
    e = rng.standard_exponential((n, d))
    bad = e <= 0.0
    while bad.any():
        e[bad] = rng.standard_exponential(int(bad.sum()))
        bad = e <= 0.0
    return e / e.sum(axis=1, keepdims=True)


def experiment_points(n: int, d: int, seed: int = 0) -> np.ndarray:
    """bench.py:125-127 generate_points: the (seed, DATA, d) substream."""
    return simplex_points(d, n, substream(seed, TAG_DATA, d))


class KlTables:
    """similarity.py:87-95 precompute and 101-106 batch_scores."""

    def __init__(self, points: np.ndarray):
        self.points = np.asarray(points, dtype=np.float64)
        self.log = np.log(self.points)
        self.xlogx = np.einsum("ij,ij->i", self.points, self.log)

    def scores(self, x: int, ids: np.ndarray | None = None) -> np.ndarray:
        rows = self.log if ids is None else self.log[ids]
        return self.xlogx[x] - np.einsum("ij,j->i", rows, self.points[x])


# --------------------------------------------------------------------------
# initial digraph — descent.py:163-213


def random_kout_draws(n: int, k: int, rng: np.random.Generator) -> np.ndarray:
    """descent.py:189-212: K distinct non-self targets per row (unsorted)."""
    if n <= k:
        raise ValueError(f"need n > k, got n={n}, k={k}")
    me = np.arange(n, dtype=np.int64)[:, None]
    if n - 1 > 2 * k * k:
        t = rng.integers(0, n - 1, size=(n, k), dtype=np.int64)
        t += t >= me
        while True:
            s = np.sort(t, axis=1)
            dup_rows = np.flatnonzero((s[:, 1:] == s[:, :-1]).any(axis=1))
            if dup_rows.size == 0:
                return t
            fresh = rng.integers(0, n - 1, size=(dup_rows.size, k), dtype=np.int64)
            fresh += fresh >= dup_rows[:, None]
            t[dup_rows] = fresh
    t = np.empty((n, k), dtype=np.int64)
    for x in range(n):
        row = rng.permutation(n - 1)[:k]
        t[x] = row + (row >= x)
    return t


def order_rows(tab: KlTables, draws: np.ndarray) -> np.ndarray:
    """descent.py:163-170: each row stably sorted by its anchor's scores."""
    out = np.empty_like(draws)
    for x in range(draws.shape[0]):
        out[x] = draws[x][np.argsort(tab.scores(x, draws[x]), kind="stable")]
    return out


# --------------------------------------------------------------------------
# one round — descent.py:151-160, 230-242, 262-314, 317-338


def cofriend_csr(friends: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """descent.py:151-160: CSR transpose; sources ascending within a target."""
    n, k = friends.shape
    flat = friends.reshape(-1)
    perm = np.argsort(flat, kind="stable")
    src = (np.arange(n * k, dtype=np.int64) // k)[perm]
    ptr = np.concatenate(([0], np.cumsum(np.bincount(flat, minlength=n)))).astype(np.int64)
    return ptr, src


def join_row(x: int, friends: np.ndarray, ptr: np.ndarray, src: np.ndarray, tab: KlTables):
    """descent.py:230-242: best K of unique(F + C + F(F) + F(C)) minus x.

    Returns (row, |U|, scores of row)."""
    k = friends.shape[1]
    f = friends[x]
    c = src[ptr[x] : ptr[x + 1]]
    u = np.unique(np.concatenate((f, c, friends[f].reshape(-1), friends[c].reshape(-1))))
    u = u[u != x]
    s = tab.scores(x, u)
    best = np.argsort(s, kind="stable")[:k]
    return u[best], int(u.size), s[best]


def local_join(friends: np.ndarray, tab: KlTables, rows: range | None = None):
    """descent.py:262-279 + 291-302: the new table, comparisons, changed."""
    n, k = friends.shape
    ptr, src = cofriend_csr(friends)
    rows = range(n) if rows is None else rows
    new = np.empty((len(rows), k), dtype=np.int64)
    comps = changed = 0
    for i, x in enumerate(rows):
        row, m, _ = join_row(x, friends, ptr, src, tab)
        comps += m
        changed += int(not np.array_equal(row, friends[x]))
        new[i] = row
    return new, comps, changed


def fcc_draws(n: int, k: int, samples: int, rng: np.random.Generator):
    """descent.py:330-333: sample anchors and an ordered pair of distinct slots."""
    xs = rng.integers(0, n, size=samples)
    i = rng.integers(0, k, size=samples)
    j = rng.integers(0, k - 1, size=samples)
    j = j + (j >= i)
    return xs, i, j


def fcc_count(friends: np.ndarray, xs, i, j) -> int:
    """descent.py:334-337: number of sampled friend pairs that are adjacent."""
    y = friends[xs, i]
    z = friends[xs, j]
    hit = (friends[z] == y[:, None]).any(axis=1) | (friends[y] == z[:, None]).any(axis=1)
    return int(hit.sum())


def fcc_rate(friends: np.ndarray, samples: int, seed: int, round_index: int) -> tuple[int, float]:
    """descent.py:305 + 317-338: (count, rate) with the (seed, FCC, round) stream."""
    n, k = friends.shape
    if k < 2 or samples < 1:
        raise ValueError("fcc needs k >= 2 and samples >= 1")
    xs, i, j = fcc_draws(n, k, samples, substream(seed, TAG_FCC, round_index))
    cnt = fcc_count(friends, xs, i, j)
    # bool mean == exact count / samples (one correctly rounded division)
    return cnt, cnt / samples


# --------------------------------------------------------------------------
# driver — descent.py:341-373


def descend(points: np.ndarray, k: int, seed: int = 0, samples: int = 1000, max_rounds: int | None = None,
            on_round=None):
    """descent.py:341-362 with stop_on_fixed_point=False (i.e. run()).

    Returns (final table int64, list of per-round dicts)."""
    tab = KlTables(points)
    n = points.shape[0]
    table = order_rows(tab, random_kout_draws(n, k, substream(seed, TAG_INIT)))
    hist = []
    for r in range(1, round_cap(n, k, max_rounds) + 1):
        new, comps, changed = local_join(table, tab)
        cnt, rate = fcc_rate(new, samples, seed, r)
        hist.append({"round": r, "comparisons": comps, "changed": changed, "fcc_count": cnt, "fcc": rate})
        if on_round is not None:
            on_round(r, table, new)
        table = new
        if len(hist) >= 2 and hist[-1]["fcc"] <= hist[-2]["fcc"]:
            break
    return table, hist


# --------------------------------------------------------------------------
# exact neighbours and recall — evaluation.py:53-137


def smallest_k(s: np.ndarray, k: int) -> np.ndarray:
    """evaluation.py:53-69: the k smallest by (score, index)."""
    return np.argsort(s, kind="stable")[:k]


def exact_rows(tab: KlTables, queries: np.ndarray, k: int) -> np.ndarray:
    """evaluation.py:86-90 loop body for the given query ids."""
    out = np.empty((len(queries), k), dtype=np.int64)
    for i, x in enumerate(queries):
        s = tab.scores(int(x)).copy()
        s[x] = np.inf
        out[i] = smallest_k(s, k)
    return out


def recall_of(approx: np.ndarray, exact: np.ndarray, queries: np.ndarray) -> float:
    """evaluation.py:111-132 with exact rows given per query (row i <-> queries[i])."""
    hits = sum(np.intersect1d(approx[int(x)], exact[i]).size for i, x in enumerate(queries))
    return hits / (len(queries) * exact.shape[1])


def recall_sample(n: int, seed: int, size: int) -> np.ndarray:
    """evaluation.py:135-137: ids drawn without replacement from the RECALL stream."""
    return substream(seed, TAG_RECALL).choice(n, size=min(size, n), replace=False)
