"""Determinism probe: consecutive run() calls on one ranking system."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2202_00517_b200 as b2

def sha(a): return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()[:12]
pts = b2.sample_simplex_uniform(5, 500, 23)
ds = b2.Dataset(pts)
cfg = b2.DescentConfig(k=6, seed=23)
mode = sys.argv[1] if len(sys.argv) > 1 else "plain"
rs = b2.KlRankingSystem(pts, validate=False)
for i in range(3):
    if mode == "empty_cache":
        torch.cuda.empty_cache()
    if mode == "fresh_rs":
        rs = b2.KlRankingSystem(pts, validate=False)
    f, h = b2.run(ds, rs, cfg)
    print(mode, i, sha(f), [[s.fcc, s.comparisons, s.changed_friend_sets] for s in h], flush=True)
