"""Candidate-list lengths of the tensor-core exact K-NN screen (knnd_exact_knn):
how many candidates per query fall inside theta_q (band included), and the
time of one call.  usage: python tools/exact_counts.py n d k queries cap"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2202_00517_b200 as b2
from paper_2202_00517_b200 import evaluation as ev
from oracle import port

n, d, k, nq, cap = (int(a) for a in sys.argv[1:6])
pts = port.experiment_points(n, d, 0)
rs = b2.KlRankingSystem(pts, validate=False)
tabs = rs.device_tables()
q = torch.from_numpy(port.recall_sample(n, 0, nq).astype(np.int32)).cuda()
ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ev._exact_call(tabs, q, k, cap, ids, None, cnt)
    torch.cuda.synchronize(); t1 = time.perf_counter()
c = cnt.cpu().numpy()
print(f"n={n} d={d} K={k} nq={nq} cap={cap}: {t1 - t0:.4f} s; count min {c.min()} median {np.median(c)} "
      f"mean {c.mean():.1f} p99 {np.percentile(c, 99)} max {c.max()} over-cap {(c > cap).sum()}")
