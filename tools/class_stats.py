"""Per-size-class anchor / comparison counts per round at a BASELINE config
(pairs with an ncu launch list of the same run for per-class throughput)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2202_00517_b200 as b2
from oracle import port

n, d, k = (int(a) for a in sys.argv[1:4])
pts = port.experiment_points(n, d, 0)
rs = b2.KlRankingSystem(pts, validate=False)
cfg = b2.DescentConfig(k=k, seed=0)
st = b2.init_random_kout(b2.Dataset(pts), rs, cfg, b2.derive_rng(0, 2))
tabs = rs.device_tables()
K1 = k + 1
lims = [int(x) for x in (sys.argv[4].split(",") if len(sys.argv) > 4 else ["1024", "2048", "8192"])]
hist = []
for r in range(cfg.resolved_max_rounds(n)):
    c = np.diff(st._csr.indptr.cpu().numpy())
    P = (k + c) * K1
    uc = torch.empty(n, dtype=torch.int32, device=tabs.device)
    out = torch.empty((n, k), dtype=torch.int32, device=tabs.device)
    tally = torch.zeros(4, dtype=torch.int64, device=tabs.device)
    st._engine.ops.join(tabs, st._table, n, k, st._csr, st._max_indeg, out, tally, None, uc)
    U = uc.cpu().numpy()
    cls = np.searchsorted(np.array(lims), P, side="left")  # class i: P <= lims[i]
    line = f"r{r+1}: "
    for i in range(len(lims) + 1):
        m = cls == i
        line += f"[c{i}: {m.sum()} anchors, U {U[m].sum()/1e6:.1f}M, P {P[m].sum()/1e6:.1f}M] "
    print(line, flush=True)
    st, s = b2.run_round(st, rs, cfg)
    hist.append(s)
    if len(hist) >= 2 and hist[-1].fcc <= hist[-2].fcc:
        break
