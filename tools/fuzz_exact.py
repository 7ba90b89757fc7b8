"""Randomised parity campaign for the tensor-core exact K-NN: exact_rows on the
device against the C brute force (pinned to evaluation.py's exact_knn body).
usage: python tools/fuzz_exact.py COUNT SEED"""
import os
import sys
import time
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2202_00517_b200 as b2  # noqa: E402
from oracle import native, port  # noqa: E402

count, seed0 = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed0)
bad = 0
t0 = time.time()
for i in range(count):
    k = int(rng.integers(1, 65))
    n = int(rng.integers(k + 1, int(rng.choice([300, 5000, 50000, 200000]))))
    metric = "kl" if rng.random() < 0.6 else "l2"
    d = int(rng.integers(1, 96 if metric == "kl" else 94))
    dup = rng.random() < 0.3
    r = np.random.default_rng(seed0 * 1000 + i)
    try:
        if metric == "kl":
            pts = port.simplex_points(d, n, r)
            if rng.random() < 0.2:  # non-simplex positive data: the Cauchy-Schwarz band
                pts = pts * r.uniform(0.5, 20.0)
            if dup:
                m = max(1, int(n * r.uniform(0.001, 0.05)))
                pts[n - m:] = pts[int(r.integers(0, n - m))]
            rs = b2.KlRankingSystem(pts, validate=False)
            tab = native.Tables(pts)
        else:
            pts = r.normal(size=(n, d)) * r.uniform(0.1, 5.0) + r.uniform(-50, 50)
            if dup:
                m = max(1, int(n * r.uniform(0.001, 0.05)))
                pts[n - m:] = pts[int(r.integers(0, n - m))]
            rs = b2.EuclideanRankingSystem(pts)
            tab = native.L2Tables(pts)
        q = np.sort(r.choice(n, size=min(n, int(r.integers(1, 3000))), replace=False))
        got = b2.exact_rows(rs, q, k)
        want = native.exact_rows(tab, q, k).astype(np.int64)
        ok = np.array_equal(got, want)
    except Exception:
        ok = False
        traceback.print_exc()
    tag = f"case {i}: n={n} d={d} k={k} {metric}{' dup' if dup else ''} q={len(q) if 'q' in dir() else '?'}"
    if not ok:
        bad += 1
        print("MISMATCH", tag, flush=True)
    elif i % 25 == 0:
        print("ok", tag, f"{time.time() - t0:.0f}s", flush=True)
print(f"done: {count} cases, {bad} mismatches, {time.time() - t0:.0f}s", flush=True)
