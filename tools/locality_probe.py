"""How much would point locality buy?  Runs the descent on the same points in
their generated (random) order and relabelled by a coarse locality key (the
indices of the largest coordinates, lexicographic), and prints comparisons/s
of each.  The relabelled run is a different instance (its ids and therefore
its init draws differ), so only the rates are comparable.
Usage: python tools/locality_probe.py n d k [top]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_00517_b200 as b2  # noqa: E402
from oracle import port  # noqa: E402

n, d, k = (int(a) for a in sys.argv[1:4])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 3
pts0 = port.experiment_points(n, d, 0)
order = np.argsort(-pts0, axis=1)[:, :top]
key = np.zeros(n, dtype=np.int64)
for j in range(top):
    key = key * d + order[:, j]
perm = np.argsort(key, kind="stable")
cfg = b2.DescentConfig(k=k, seed=0)
for name, pts in (("generated", pts0), (f"top{top}-sorted", np.ascontiguousarray(pts0[perm]))):
    rs = b2.KlRankingSystem(pts, validate=False)
    best = None
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = b2.init_random_kout(b2.Dataset(pts), rs, cfg, b2.derive_rng(0, 2))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        hist = []
        for r in range(cfg.resolved_max_rounds(n)):
            st, s = b2.run_round(st, rs, cfg)
            hist.append(s)
            if len(hist) >= 2 and hist[-1].fcc <= hist[-2].fcc:
                break
        t2 = time.perf_counter()
        tot = sum(h.comparisons for h in hist)
        rate = tot / (t2 - t1)
        best = max(best or 0, rate)
        print(f"{name} rep {rep}: rounds {len(hist)} {t2 - t1:.4f}s comps {tot} -> {rate:.3e}/s", flush=True)
    print(f"== {name}: best {best:.3e}/s", flush=True)
