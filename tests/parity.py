"""Parity helpers shared by the GPU tests (checker side: uses oracle/)."""

from __future__ import annotations

import hashlib

import numpy as np

from oracle import native

TIE_REL = 1e-6  # BASELINE north_star: rows bit-exact except ties within 1e-6 relative
KL_REL = 1e-5  # KL values within 1e-5 relative of the fp64 reference


def sha_i32(t) -> str:
    return hashlib.sha256(np.ascontiguousarray(t, dtype="<i4").tobytes()).hexdigest()


def oracle_scores(tab: native.Tables, x: int, ids) -> np.ndarray:
    ids = np.asarray(ids, dtype=np.int64)
    return tab.xlogx[x] - np.einsum("ij,j->i", tab.log[ids], tab.points[x])


def tie_aware_diff(tab: native.Tables, expect: np.ndarray, got: np.ndarray, anchors=None) -> dict:
    """Compare two (m, K) tables row by row.  Returns counts; every differing
    slot must swap ids whose fp64 scores tie within TIE_REL (else 'violations')."""
    expect = np.asarray(expect)
    got = np.asarray(got)
    anchors = np.arange(expect.shape[0]) if anchors is None else np.asarray(anchors)
    rows = np.nonzero((expect != got).any(axis=1))[0]
    violations = []
    member_diff = 0
    for r in rows:
        x = int(anchors[r])
        e, g = expect[r], got[r]
        if set(e.tolist()) != set(g.tolist()):
            member_diff += 1
        se = oracle_scores(tab, x, e)
        sg = oracle_scores(tab, x, g)
        for i in np.nonzero(e != g)[0]:
            scale = max(abs(se[i]), abs(sg[i]), 1e-300)
            if abs(se[i] - sg[i]) > TIE_REL * scale:
                violations.append((x, int(i), int(e[i]), int(g[i]), float(se[i]), float(sg[i])))
    return {"rows": int(rows.size), "members": member_diff, "violations": violations}
