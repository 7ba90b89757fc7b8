"""CSR build timing at n, K (random K-out table): python tools/csr_probe.py [n k reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2202_00517_b200 as b2
from paper_2202_00517_b200.engine import Engine

n, k = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (1_000_000, 20)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
eng = Engine(n, k, torch.device("cuda", 0))
t = eng.upload_table(b2.random_kout_draws(n, k, np.random.default_rng(1)))
for _ in range(2):
    eng.ops.csr(t, n, k, 0, n, eng._stats32[9:10])
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    eng.ops.csr(t, n, k, 0, n, eng._stats32[9:10])
e1.record(); torch.cuda.synchronize()
print(f"csr n={n} k={k}: {e0.elapsed_time(e1) / reps:.3f} ms per build")
