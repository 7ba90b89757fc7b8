"""Break down the end-to-end run() time at a BASELINE config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2202_00517_b200 as b2
from paper_2202_00517_b200.descent import draw_fcc_schedule, _to_device, descend_resident, device_random_kout
from paper_2202_00517_b200.engine import Engine

n, d, k = (int(a) for a in sys.argv[1:4])
pts = b2.sample_simplex_uniform(d, n, b2.derive_rng(0, 1, d))
cfg = b2.DescentConfig(k=k, seed=0)
def t():
    torch.cuda.synchronize(); return time.perf_counter()
for rep in range(4):
    T = {}
    t0 = t()
    rs = b2.KlRankingSystem(pts, validate=False); t1 = t(); T["KlRankingSystem()"] = t1 - t0
    tabs = rs.device_tables(); t2 = t(); T["device tables"] = t2 - t1
    eng = Engine(n, k, tabs.device); table = eng.alloc_table(); t3 = t(); T["engine+alloc"] = t3 - t2
    device_random_kout(eng, n, k, b2.derive_rng(0, 2), table); t4 = t(); T["device draws"] = t4 - t3
    R = cfg.resolved_max_rounds(n)
    smp = _to_device(draw_fcc_schedule(n, k, cfg, R), tabs.device); t5 = t(); T["fcc schedule"] = t5 - t4
    st, hist = descend_resident(eng, tabs, table, smp, 1000, R); t6 = t(); T["device descent"] = t6 - t5
    f = st.friends; t7 = t(); T["download"] = t7 - t6
    T["total"] = t7 - t0
    print(rep, {k_: round(v * 1e3, 1) for k_, v in T.items()}, flush=True)
    t8 = t(); rs2 = b2.KlRankingSystem(pts, validate=False); fr, h = b2.run(b2.Dataset(pts), rs2, cfg); print("  run()", round((t() - t8) * 1e3, 1), "ms", flush=True)
