"""Time the GPU exact K-NN (knnd_exact_knn) at a BASELINE config:
usage: python tools/exact_probe.py n d k [queries]  (queries: 'all' or a count)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2202_00517_b200 as b2
from oracle import port

n, d, k = (int(a) for a in sys.argv[1:4])
which = sys.argv[4] if len(sys.argv) > 4 else "10000"
pts = port.experiment_points(n, d, 0)
rs = b2.KlRankingSystem(pts, validate=False)
q = np.arange(n) if which == "all" else port.recall_sample(n, 0, int(which))
b2.evaluation.exact_rows_device(rs, q[:1000], k)  # warm-up
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ids = b2.evaluation.exact_rows_device(rs, q, k)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    pairs = len(q) * (n - 1)
    print(f"rep {rep}: {len(q)} queries x {n} points: {t1 - t0:.3f} s, {pairs / (t1 - t0):.3e} scored pairs/s "
          f"({2 * pairs * d / (t1 - t0) / 1e12:.1f} TFLOP/s fp32 per sweep x2 sweeps)", flush=True)
