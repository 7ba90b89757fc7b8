"""Ground truth and recall (reference evaluation.py:36-137) with the exact
K-NN computed on the GPU (knnd_exact_knn).

``exact_knn`` / ``ExactKnnGraph`` / ``recall`` / ``uniform_recall_sample`` keep
the reference's names, arguments and results: row x of the exact graph is the
K smallest (fp64 score, id) over every other point (evaluation.py:83-90, the
``_smallest_k`` order of evaluation.py:53-71).  ``exact_rows`` is the same
computation for a subset of anchors — what a sampled recall at n = 1M needs.
The KL and Euclidean ranking systems are accelerated (no CPU fallback); the
metrizability checker (evaluation.py:140-) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Mapping, Sequence

import numpy as np
import torch

from . import _lib
from .core import ConfigError, Dataset, ItemId
from .descent import STREAM_RECALL, derive_rng
from .engine import workspace
from .similarity import device_tables_for

_QCTA = 256  # queries per CTA of the tensor-core screen (exact.cu TC_Q)


def _batch(device) -> int:
    """Queries per device call: whole waves of the screen's CTAs (one per SM),
    four waves per call (bounds the candidate lists to ~600 MB at cap 1024)."""
    return torch.cuda.get_device_properties(device).multi_processor_count * _QCTA * 4
_CAP = 1024  # initial candidate-list capacity per query (rows that overflow are rerun: a whole extra pass)


@dataclass
class ExactKnnGraph:
    """True K nearest neighbors of every item, nearest first (evaluation.py:36-50)."""

    neighbors: np.ndarray  # (n, K) ids

    @property
    def n(self) -> int:
        return self.neighbors.shape[0]

    @property
    def k(self) -> int:
        return self.neighbors.shape[1]

    def of(self, x: ItemId) -> np.ndarray:
        return self.neighbors[x]


def _exact_call(tabs, q: torch.Tensor, k: int, cap: int, ids: torch.Tensor, scores: torch.Tensor | None,
                count: torch.Tensor) -> None:
    nbytes = _lib.load().knnd_exact_knn_workspace_bytes(tabs.n, tabs.ld, q.numel(), cap)
    ws = workspace(nbytes, tabs.device)
    tabs.exact(q, k, cap, ids, scores, count, ws, torch.cuda.current_stream(tabs.device).cuda_stream)


def exact_rows_device(rs, queries, k: int, device=None, with_scores: bool = False):
    """Exact rows of the given anchors, left on the device: int32 (q, K) ids
    (and fp64 scores when asked)."""
    tabs = device_tables_for(rs, device)
    n = tabs.n
    if n <= k:
        raise ConfigError(f"need n > k, got n={n}, k={k}")
    qh = np.asarray(queries, dtype=np.int64).reshape(-1)
    if qh.size and (qh.min() < 0 or qh.max() >= n):
        raise ValueError("query ids must lie in [0, n)")
    q_all = torch.from_numpy(qh.astype(np.int32)).to(tabs.device)
    ids = torch.empty((qh.size, k), dtype=torch.int32, device=tabs.device)
    scores = torch.empty((qh.size, k), dtype=torch.float64, device=tabs.device) if with_scores else None
    step = _batch(tabs.device)
    for lo in range(0, qh.size, step):
        hi = min(lo + step, qh.size)
        q = q_all[lo:hi]
        count = torch.empty(hi - lo, dtype=torch.int32, device=tabs.device)
        _exact_call(tabs, q, k, _CAP, ids[lo:hi], scores[lo:hi] if with_scores else None, count)
        cap, sel, cnt = _CAP, torch.arange(hi - lo, device=tabs.device), count
        over = torch.nonzero(cnt > cap).flatten()
        while over.numel():  # rare: many candidates inside the error band (e.g. duplicate points)
            cap = max(int(cnt[over].max().item()), 2 * cap)
            sel = sel[over]
            q2 = q[sel].contiguous()
            ids2 = torch.empty((q2.numel(), k), dtype=torch.int32, device=tabs.device)
            sc2 = torch.empty((q2.numel(), k), dtype=torch.float64, device=tabs.device) if with_scores else None
            cnt = torch.empty(q2.numel(), dtype=torch.int32, device=tabs.device)
            _exact_call(tabs, q2, k, cap, ids2, sc2, cnt)
            ok = cnt <= cap  # rows written by this call
            ids[lo:hi][sel[ok]] = ids2[ok]
            if with_scores:
                scores[lo:hi][sel[ok]] = sc2[ok]
            over = torch.nonzero(~ok).flatten()
    return (ids, scores) if with_scores else ids


def exact_rows(rs, queries, k: int, device=None) -> np.ndarray:
    """(len(queries), K) int64: row a = the exact K nearest of queries[a]
    (evaluation.py:86-90 for each sampled anchor)."""
    return exact_rows_device(rs, queries, k, device).cpu().numpy().astype(np.int64)


def exact_knn(dataset: Dataset, rs, k: int, workers: int = 1) -> ExactKnnGraph:
    """evaluation.py:74-108 — the exact K-NN digraph of every item (on the GPU;
    ``workers`` is accepted for signature compatibility and changes nothing,
    as in the reference)."""
    n = len(dataset)
    if n <= k:
        raise ConfigError(f"need n > k, got n={n}, k={k}")
    return ExactKnnGraph(exact_rows(rs, np.arange(n), k))


def recall(
    approx: np.ndarray | Mapping[int, Iterable[int]],
    exact: ExactKnnGraph,
    sample_ids: Sequence[int] | np.ndarray,
) -> float:
    """evaluation.py:111-132 — mean fraction of true K nearest neighbours
    present in the approximate sets."""
    sample = np.asarray(sample_ids)
    if sample.size == 0:
        raise ValueError("sample_ids must be nonempty")
    if isinstance(approx, Mapping):
        rows = {x: np.fromiter(approx[int(x)], dtype=np.int64) for x in sample}
        widths = {r.size for r in rows.values()}
        if widths != {exact.k}:
            raise ValueError(f"approximate sets have sizes {sorted(widths)}, exact K is {exact.k}")
        get = rows.__getitem__
    else:
        approx = np.asarray(approx)
        if approx.shape[1] != exact.k:
            raise ValueError(f"K mismatch: approximate {approx.shape[1]} vs exact {exact.k}")
        get = approx.__getitem__
    hits = sum(np.intersect1d(get(x), exact.neighbors[x]).size for x in sample)
    return hits / (sample.size * exact.k)


def sampled_recall(approx: np.ndarray, rs, sample_ids, device=None) -> float:
    """recall of `approx` over `sample_ids` with the exact rows of just those
    anchors computed on the GPU (the protocol for n >= 1M)."""
    sample = np.asarray(sample_ids, dtype=np.int64)
    if sample.size == 0:
        raise ValueError("sample_ids must be nonempty")
    approx = np.asarray(approx)
    k = approx.shape[1]
    ex = exact_rows(rs, sample, k, device)
    hits = sum(np.intersect1d(approx[x], ex[i]).size for i, x in enumerate(sample))
    return hits / (sample.size * k)


def uniform_recall_sample(n: int, seed: int, size: int = 6) -> np.ndarray:
    """evaluation.py:135-137 — size ids drawn uniformly without replacement."""
    return derive_rng(seed, STREAM_RECALL).choice(n, size=min(size, n), replace=False)
