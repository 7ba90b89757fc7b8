"""Replay one case of tools/fuzz.py (same draws) and report where the device and the oracle differ.
usage: python tools/fuzz_repro.py SEED0 CASE [KNND_Q23 value]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
seed0, case = int(sys.argv[1]), int(sys.argv[2])
force = sys.argv[3] if len(sys.argv) > 3 else None
import paper_2202_00517_b200 as b2
from oracle import native, port

rng = np.random.default_rng(seed0)
for i in range(case + 1):
    k = int(rng.choice([2, 3, 4, 5, 7, 8, 10, 12, 16, 20, 24, 30, 31, 32, 33, 40, 48, 63, 64]))
    n = int(rng.integers(k + 2, int(rng.choice([200, 5000, 60000, 200000]))))
    d = int(rng.integers(1, 70))
    metric = "kl" if rng.random() < 0.7 else "l2"
    q23 = rng.random() < 0.6
    dup = rng.random() < 0.3
os.environ["KNND_Q23"] = force if force is not None else ("1" if q23 else "0")
print(f"case {case}: n={n} d={d} k={k} {metric} q23={os.environ['KNND_Q23']} dup={dup}")
r = np.random.default_rng(seed0 * 1000 + case)
assert metric == "kl"
pts = port.simplex_points(d, n, r)
if dup:
    m = max(1, int(n * r.uniform(0.01, 0.3)))
    src = int(r.integers(0, n - m))
    pts[n - m:] = pts[src]
    print("dup block", n - m, "..", n, "copies of", src)
rs = b2.KlRankingSystem(pts, validate=False)
tab = native.Tables(pts)
s = int(r.integers(0, 1 << 30))
cfg = b2.DescentConfig(k=k, seed=s)
st = b2.init_random_kout(b2.Dataset(pts), rs, cfg, b2.derive_rng(s, 2))
cur = native.sort_rows(tab, port.random_kout_draws(n, k, port.substream(s, port.TAG_INIT)))
assert np.array_equal(st.friends, cur), "init differs"
for rnd in range(1, 12):
    st, stats = b2.run_round(st, rs, cfg)
    rows, _, uc, comps, changed = native.local_join(tab, cur)
    got = st.friends
    bad = np.nonzero((got != rows).any(axis=1))[0]
    print(f"round {rnd}: comps {stats.comparisons} vs {comps}, changed {stats.changed_friend_sets} vs {changed}, rows differing {bad.size}")
    if bad.size:
        import torch
        indeg = np.bincount(cur.ravel(), minlength=n)
        # the same join again on the oracle's input, with |U| per anchor
        st0 = b2.KnnState(cur)
        dev = st0.device
        out = torch.empty((n, k), dtype=torch.int32, device=dev)
        ucd = torch.empty(n, dtype=torch.int32, device=dev)
        tally = torch.zeros(4, dtype=torch.int64, device=dev)
        st0._engine.ops.join(rs.device_tables(), st0._table, n, k, st0._csr, st0._max_indeg, out, tally, None, ucd)
        ucd = ucd.cpu().numpy()
        wrongu = np.nonzero(ucd != uc)[0]
        print("  max indeg", indeg.max(), "anchors with wrong |U|:", wrongu.size, [(int(x), int(indeg[x]), int(ucd[x]), int(uc[x])) for x in wrongu[:8]])
        P = (k + indeg) * (k + 1)
        print("  P of wrong-row anchors", [int(P[x]) for x in bad[:8]], " P of wrong-|U| anchors", sorted(set(int(P[x]) for x in wrongu))[:10])
        # a differing row is within the parity contract when it is a reordering of candidates
        # whose fp64 scores tie within 1e-6 relative of the cross entropy (the reference's
        # einsum and the device's FMA chain round differently at ~1e-16)
        ties = 0
        for x in bad:
            if sorted(got[x]) == sorted(rows[x]):
                sc = rs.batch_scores(int(x), rows[x].astype(np.int64))
                ce = float(-(pts[x] * np.log(pts[rows[x][0]])).sum())
                pos = [i for i in range(k) if got[x][i] != rows[x][i]]
                if np.ptp(sc[pos]) <= 1e-6 * max(abs(ce), 1e-300):
                    ties += 1
        print(f"  differing rows that only reorder ties within 1e-6 relative: {ties} of {bad.size}")
        for x in bad[:6]:
            print("  anchor", x, "indeg", indeg[x], "|U|", uc[x], "got", got[x], "want", rows[x],
                  "kl got", [float(rs.batch_scores(int(x), np.array([g]))[0]) for g in got[x]],
                  "kl want", [float(rs.batch_scores(int(x), np.array([g]))[0]) for g in rows[x]])
        break
    cur = rows
