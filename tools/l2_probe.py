"""Time the squared-Euclidean descent (EuclideanRankingSystem) at n, d, K on
seeded Gaussian vectors: per-round join time and comparisons/s, plus recall on
a 10k sample with the GPU exact rows."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2202_00517_b200 as b2

n, d, k = (int(a) for a in sys.argv[1:4])
v = np.random.default_rng(0).standard_normal((n, d))
rs = b2.EuclideanRankingSystem(v)
cfg = b2.DescentConfig(k=k, seed=0)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st = b2.init_random_kout(b2.Dataset(v), rs, cfg, b2.derive_rng(0, 2))
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
    jm = sum(ms for ms, _ in st._engine.join_events)
    print(f"rep {rep}: init {t1-t0:.3f}s rounds {t2-t1:.3f}s ({len(hist)} rounds) comps {tot} -> {tot/(t2-t1):.3e}/s; "
          f"join only {tot/(jm*1e-3):.3e}/s", flush=True)
sample = b2.uniform_recall_sample(n, 0, 10_000)
print("recall@K on 10k sample:", b2.sampled_recall(st.friends, rs, sample))
