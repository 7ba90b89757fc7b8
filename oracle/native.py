"""ctypes wrapper for oracle/knnd_oracle.c (TEST INFRASTRUCTURE ONLY).

Build recipe: ``gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC`` into
oracle/liboracle.so (git-ignored, travels to the GPU box with the snapshot).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "knnd_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp"
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC", SRC, "-o", tmp, "-lm"]
        subprocess.run(cmd, check=True, capture_output=True, text=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        i64, i32 = C.c_int64, C.c_int
        L.oracle_transpose.argtypes = [P, i64, i32, P, P]
        L.oracle_transpose.restype = None
        L.oracle_local_join.argtypes = [P, P, P, i64, i32, i32, P, i32, P, P, P, i64, P, P, P, P, i32]
        L.oracle_local_join.restype = i32
        L.oracle_fcc.argtypes = [P, i64, i32, P, P, P, i64]
        L.oracle_fcc.restype = C.c_int32
        L.oracle_sort_rows.argtypes = [P, P, P, i64, i32, i32, i32, P, P, i32]
        L.oracle_sort_rows.restype = None
        L.oracle_exact_rows.argtypes = [P, P, P, i64, i32, i32, i32, P, i64, P, i32]
        L.oracle_exact_rows.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Tables:
    """fp64 points, log and xlogx as similarity.py:91-93 computes them."""

    metric = 0

    def __init__(self, points: np.ndarray):
        self.points = _c(points, np.float64)
        self.log = np.log(self.points)
        self.xlogx = np.einsum("ij,ij->i", self.points, self.log)
        self.n, self.d = self.points.shape


class L2Tables:
    """Squared-Euclidean scoring (similarity.py:119-140): the vectors and their
    squared norms (einsum, similarity.py:128) in the slots the C oracle reads."""

    metric = 1

    def __init__(self, vectors: np.ndarray):
        self.points = _c(vectors, np.float64)
        self.log = self.points
        self.xlogx = np.einsum("ij,ij->i", self.points, self.points)
        self.n, self.d = self.points.shape


def transpose(friends: np.ndarray):
    F = _c(friends, np.int32)
    n, k = F.shape
    ptr = np.empty(n + 1, np.int64)
    idx = np.empty(n * k, np.int32)
    lib().oracle_transpose(_p(F), n, k, _p(ptr), _p(idx))
    return ptr, idx


def local_join(tab: Tables, friends: np.ndarray, anchors: np.ndarray | None = None, csr=None, threads: int = 0):
    """Returns (rows int32 (na,K), scores f64 (na,K), ucount int32 (na,), comparisons, changed)."""
    F = _c(friends, np.int32)
    n, k = F.shape
    ptr, idx = csr if csr is not None else transpose(F)
    ptr = _c(ptr, np.int64)
    idx = _c(idx, np.int32)
    anchors = np.arange(n, dtype=np.int64) if anchors is None else _c(anchors, np.int64)
    na = anchors.size
    out = np.empty((na, k), np.int32)
    kl = np.empty((na, k), np.float64)
    uc = np.empty(na, np.int32)
    tally = np.zeros(2, np.int64)
    rc = lib().oracle_local_join(_p(tab.points), _p(tab.log), _p(tab.xlogx), n, tab.d, tab.metric, _p(F), k, _p(ptr), _p(idx),
                                 _p(anchors), na, _p(out), _p(kl), _p(uc), _p(tally), threads)
    if rc != 0:
        raise ValueError("oracle_local_join: unsupported K")
    return out, kl, uc, int(tally[0]), int(tally[1])


def fcc_count(friends: np.ndarray, xs, i, j) -> int:
    F = _c(friends, np.int32)
    n, k = F.shape
    xs, i, j = (_c(a, np.int64) for a in (xs, i, j))
    return int(lib().oracle_fcc(_p(F), n, k, _p(xs), _p(i), _p(j), xs.size))


def sort_rows(tab: Tables, draws: np.ndarray, threads: int = 0) -> np.ndarray:
    D = _c(draws, np.int32)
    n, k = D.shape
    out = np.empty_like(D)
    lib().oracle_sort_rows(_p(tab.points), _p(tab.log), _p(tab.xlogx), n, tab.d, tab.metric, k, _p(D), _p(out), threads)
    return out


def exact_rows(tab: Tables, queries: np.ndarray, k: int, threads: int = 0) -> np.ndarray:
    q = _c(queries, np.int64)
    out = np.empty((q.size, k), np.int32)
    lib().oracle_exact_rows(_p(tab.points), _p(tab.log), _p(tab.xlogx), tab.n, tab.d, tab.metric, k, _p(q), q.size, _p(out),
                            threads)
    return out


def descend(tab: Tables, init_table: np.ndarray, seed: int, samples: int, max_rounds: int, on_round=None,
            threads: int = 0):
    """The run loop (descent.py:341-362) over the C local join.  FCC draws use
    the reference's stream (descent.py:305, 330-333) via oracle.port."""
    from . import port

    table = _c(init_table, np.int32)
    n, k = table.shape
    hist = []
    for r in range(1, max_rounds + 1):
        new, _, _, comps, changed = local_join(tab, table, threads=threads)
        xs, i, j = port.fcc_draws(n, k, samples, port.substream(seed, port.TAG_FCC, r))
        cnt = fcc_count(new, xs, i, j)
        hist.append({"round": r, "comparisons": comps, "changed": changed, "fcc_count": cnt, "fcc": cnt / samples})
        if on_round is not None:
            on_round(r, table, new)
        table = new
        if len(hist) >= 2 and hist[-1]["fcc"] <= hist[-2]["fcc"]:
            break
    return table, hist
