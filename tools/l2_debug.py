"""Debug: one L2 round on a golden case, GPU rows vs the C oracle's."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np
import paper_2202_00517_b200 as b2
from oracle import native, port
from make_l2_golden import CASES, vectors

name = sys.argv[1] if len(sys.argv) > 1 else "g4"
n, d, k, seed, kind = CASES[name]
v = vectors(n, d, seed, kind)
rs = b2.EuclideanRankingSystem(v)
tab = native.L2Tables(v)
draws = port.random_kout_draws(n, k, port.substream(seed, port.TAG_INIT))
init = native.sort_rows(tab, draws)
st = b2.KnnState(init)
nxt, s = b2.run_round(st, rs, b2.DescentConfig(k=k, seed=seed))
rows, sc, uc, comps, changed = native.local_join(tab, init)
g = nxt.friends
bad = np.nonzero((g != rows).any(axis=1))[0]
print("rows differing:", bad.size, "comps", s.comparisons, comps)
for x in bad[:5]:
    print("x", x, "gpu", g[x].tolist())
    print("    ora", rows[x].tolist())
    fs = rs.batch_scores(int(x), g[x]); fo = rs.batch_scores(int(x), rows[x])
    print("    gpu scores", fs.tolist())
    print("    ora scores", fo.tolist())
    print("    oracle scores", sc[x].tolist())

# screen of anchor x over its candidate set, from the device tables
tabs = rs.device_tables()
A = tabs.anchor32.cpu().numpy(); Cc = tabs.cand32.cpu().numpy()
x = int(bad[0]) if bad.size else 5
F = init
ptr, idx = native.transpose(F)
S = list(F[x]) + list(idx[ptr[x]:ptr[x + 1]])
U = set(S)
for s_ in S:
    U |= set(F[s_].tolist())
U.discard(x)
U = np.array(sorted(U))
ce = -(A[x][None, :].astype(np.float32) * Cc[U]).sum(axis=1, dtype=np.float32)
ab = np.abs(A[x][None, :] * Cc[U]).sum(axis=1)
ex = rs.batch_scores(x, U)
o = np.lexsort((U, ex))
print("x", x, "|U|", U.size, "K-th exact", ex[o[k - 1]], "ids at K-th score:", U[ex == ex[o[k - 1]]][:10])
os_ = np.sort(ce)
print("screen K-th", os_[k - 1], "max ab", ab.max(), "ce of tied:", ce[ex == ex[o[k - 1]]][:10])
print("anchor row", A[x].tolist(), "cand rows of 102/226:", Cc[102].tolist(), Cc[226].tolist())

import torch
eng = st._engine
out = torch.empty((n, k), dtype=torch.int32, device=eng.device)
okl = torch.empty((n, k), dtype=torch.float64, device=eng.device)
ouc = torch.empty(n, dtype=torch.int32, device=eng.device)
tally = torch.zeros(4, dtype=torch.int64, device=eng.device)
eng.ops.join(tabs, st._table, n, k, st._csr, st._max_indeg, out, tally, okl, ouc)
o2 = out.cpu().numpy()
print("with out_kl: rows differing", np.nonzero((o2 != rows).any(axis=1))[0].size, "ucount equal", np.array_equal(ouc.cpu().numpy(), uc))
print("x", x, o2[x].tolist(), okl[x].cpu().numpy().tolist())
cs = np.diff(ptr)
P = (k + cs) * (k + 1)
print("P of bad rows", P[bad[:20]].tolist())
