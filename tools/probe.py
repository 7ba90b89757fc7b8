"""Quick device probe: one full run at a BASELINE config with per-round timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2202_00517_b200 as b2
from oracle import port

n, d, k = (int(a) for a in sys.argv[1:4])
pts = port.experiment_points(n, d, 0)
rs = b2.KlRankingSystem(pts, validate=False)
cfg = b2.DescentConfig(k=k, seed=0)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
for rep in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st = b2.init_random_kout(b2.Dataset(pts), rs, cfg, b2.derive_rng(0, 2))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    st._engine.join_events = []
    hist = []
    for r in range(cfg.resolved_max_rounds(n)):
        st, s = b2.run_round(st, rs, cfg)
        hist.append(s)
        if len(hist) >= 2 and hist[-1].fcc <= hist[-2].fcc:
            break
    t2 = time.perf_counter()
    tot = sum(h.comparisons for h in hist)
    print(f"rep {rep}: init {t1-t0:.3f}s rounds {t2-t1:.3f}s comps {tot} -> {tot/(t2-t1):.3e}/s")
    for h, (ms, c) in zip(hist, st._engine.join_events):
        print(f"  r{h.round_index} wall {h.wall_clock_sec*1e3:.2f}ms join {ms:.2f}ms comps {h.comparisons} "
              f"({c/ms*1e3:.3e}/s, {c*4*d/ms/1e6:.1f} GB/s) changed {h.changed_friend_sets} fcc {h.fcc}")
