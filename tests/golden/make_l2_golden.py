"""Golden trajectories of the reference with its EuclideanRankingSystem
(similarity.py:119-140) — build container only (imports /root/reference).

For each case: seeded vectors (generator below), the reference's own
init_random_kout + run_round loop exactly as rankdescent.run drives it
(descent.py:341-362), per-round sha256 / comparisons / changed / FCC count, and
the sha256 of the reference's exact_knn graph (evaluation.py:74-108).
Output: tests/golden/l2_trajectories.json.
Usage: python tests/golden/make_l2_golden.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

CASES = {
    # name: (n, d, k, seed, kind)
    "g1": (3000, 8, 10, 0, "normal"),
    "g2": (5000, 3, 8, 1, "offset"),
    "g3": (2000, 20, 20, 2, "uniform"),
    "g4": (1500, 5, 12, 3, "grid"),
    "g5": (1200, 16, 40, 4, "normal"),
}


def vectors(n: int, d: int, seed: int, kind: str) -> np.ndarray:
    """The test inputs (shared with tests/test_l2.py)."""
    g = np.random.default_rng(seed)
    if kind == "normal":
        return g.standard_normal((n, d))
    if kind == "offset":  # large norms, small distances: stresses the fp32 screen band
        return 100.0 + g.standard_normal((n, d))
    if kind == "uniform":
        return g.random((n, d))
    if kind == "grid":  # small integers: exact arithmetic, many duplicate points and exact ties
        return g.integers(0, 4, size=(n, d)).astype(np.float64)
    raise ValueError(kind)


def sha(t: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(t, dtype="<i4").tobytes()).hexdigest()


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import rankdescent as rd  # noqa: E402

    out = {}
    for name, (n, d, k, seed, kind) in CASES.items():
        v = vectors(n, d, seed, kind)
        rs = rd.EuclideanRankingSystem(v)
        ds = rd.Dataset(v)
        cfg = rd.DescentConfig(k=k, seed=seed)
        state = rd.init_random_kout(ds, rs, cfg, rd.derive_rng(seed, 2))
        rec = {"n": n, "d": d, "k": k, "seed": seed, "kind": kind, "init_sha": sha(state.friends), "rounds": []}
        hist = []
        for _ in range(cfg.resolved_max_rounds(n)):
            state, st = rd.run_round(state, rs, cfg)
            hist.append(st)
            rec["rounds"].append({"round": st.round_index, "comparisons": int(st.comparisons),
                                  "changed": int(st.changed_friend_sets),
                                  "fcc_count": int(round(st.fcc * cfg.fcc_sample_count)), "sha": sha(state.friends)})
            if len(hist) >= 2 and hist[-1].fcc <= hist[-2].fcc:
                break
        ex = rd.evaluation.exact_knn(ds, rs, k)
        rec["exact_sha"] = sha(ex.neighbors)
        rec["recall"] = rd.evaluation.recall(state.friends, ex, np.arange(n))
        out[name] = rec
        print(name, len(rec["rounds"]), "rounds, recall", rec["recall"], flush=True)
    with open(os.path.join(HERE, "l2_trajectories.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
