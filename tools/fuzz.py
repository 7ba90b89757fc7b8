"""Randomised parity campaign (not a test: many more shapes than tests/test_fuzz_gpu.py):
full device descents against the C oracle.  usage: python tools/fuzz.py COUNT SEED"""
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
    k = int(rng.choice([2, 3, 4, 5, 7, 8, 10, 12, 16, 20, 24, 30, 31, 32, 33, 40, 48, 63, 64]))
    n = int(rng.integers(k + 2, int(rng.choice([200, 5000, 60000, 200000]))))
    d = int(rng.integers(1, 70))
    metric = "kl" if rng.random() < 0.7 else "l2"
    q23 = rng.random() < 0.6  # the Q23 screen rows where the shape has them (else the fp32 rows)
    dup = rng.random() < 0.3
    os.environ["KNND_Q23"] = "1" if q23 else "0"
    r = np.random.default_rng(seed0 * 1000 + i)
    try:
        if metric == "kl":
            pts = port.simplex_points(d, n, r)
            if dup:
                m = max(1, int(n * r.uniform(0.01, 0.3)))
                pts[n - m:] = pts[int(r.integers(0, n - m))]
            rs = b2.KlRankingSystem(pts, validate=False)
            tab = native.Tables(pts)
        else:
            pts = r.normal(size=(n, d)) * r.uniform(0.1, 5.0) + r.uniform(-50, 50)
            if dup:
                m = max(1, int(n * r.uniform(0.01, 0.3)))
                pts[n - m:] = pts[int(r.integers(0, n - m))]
            rs = b2.EuclideanRankingSystem(pts)
            tab = native.L2Tables(pts)
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
    tag = f"case {i}: n={n} d={d} k={k} {metric}{' q23' if q23 else ''}{' dup' if dup else ''}"
    if not ok:
        bad += 1
        print("MISMATCH", tag, flush=True)
    elif i % 20 == 0:
        print("ok", tag, f"{time.time() - t0:.0f}s", flush=True)
print(f"done: {count} cases, {bad} mismatches, {time.time() - t0:.0f}s", flush=True)
