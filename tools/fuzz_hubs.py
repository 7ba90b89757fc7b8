"""Targeted parity campaign: small K, blocks of identical points (exact ties, in-degree hubs of
hundreds to thousands), both screens — the shapes that reach the big shared-memory classes and
the global-memory class with unusual table sizes.  usage: python tools/fuzz_hubs.py COUNT SEED"""
import os
import sys
import time
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_2202_00517_b200 as b2  # noqa: E402
from oracle import native, port  # noqa: E402

count, seed0 = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed0)
bad = 0
t0 = time.time()
for i in range(count):
    k = int(rng.choice([2, 2, 3, 3, 4, 5, 6, 8, 12, 20, 33]))
    n = int(rng.integers(max(3 * k, 500), int(rng.choice([3000, 12000, 40000]))))
    d = int(rng.choice([2, 3, 5, 6, 7, 8, 10, 12, 16, 20, 24, 50]))
    metric = "kl" if rng.random() < 0.75 else "l2"
    q23 = rng.random() < 0.6
    os.environ["KNND_Q23"] = "1" if q23 else "0"
    r = np.random.default_rng(seed0 * 1000 + i)
    blocks = int(r.integers(1, 4))  # blocks of identical points
    try:
        pts = port.simplex_points(d, n, r) if metric == "kl" else r.normal(size=(n, d)) * r.uniform(0.3, 3.0)
        at = n
        for _ in range(blocks):
            m = int(n * r.uniform(0.02, 0.25))
            at -= m
            if at <= 1:
                break
            pts[at:at + m] = pts[int(r.integers(0, at))]
        if metric == "kl":
            rs, tab = b2.KlRankingSystem(pts, validate=False), native.Tables(pts)
        else:
            rs, tab = b2.EuclideanRankingSystem(pts), native.L2Tables(pts)
        s = int(r.integers(0, 1 << 30))
        cfg = b2.DescentConfig(k=k, seed=s)
        friends, hist = b2.run(b2.Dataset(pts), rs, cfg)
        init = native.sort_rows(tab, port.random_kout_draws(n, k, port.substream(s, port.TAG_INIT)))
        final, ohist = native.descend(tab, init, s, cfg.fcc_sample_count, cfg.resolved_max_rounds(n))
        ok = ([(h.comparisons, h.changed_friend_sets, round(h.fcc * 1000)) for h in hist] ==
              [(h["comparisons"], h["changed"], h["fcc_count"]) for h in ohist]) and np.array_equal(friends, final)
    except Exception:
        ok = False
        traceback.print_exc()
    tag = f"case {i}: n={n} d={d} k={k} {metric}{' q23' if q23 else ''} blocks={blocks}"
    if not ok:
        bad += 1
        print("MISMATCH", tag, flush=True)
    elif i % 20 == 0:
        print("ok", tag, f"{time.time() - t0:.0f}s", flush=True)
print(f"done: {count} cases, {bad} mismatches, {time.time() - t0:.0f}s", flush=True)
