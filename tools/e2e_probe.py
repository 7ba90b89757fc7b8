"""Break down the end-to-end run() time at a BASELINE config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2202_00517_b200 as b2
from paper_2202_00517_b200.descent import draw_fcc_schedule, _to_device, descend_resident
from paper_2202_00517_b200.engine import Engine

n, d, k = (int(a) for a in sys.argv[1:4])
pts = b2.sample_simplex_uniform(d, n, b2.derive_rng(0, 1, d))
cfg = b2.DescentConfig(k=k, seed=0)
def t():
    torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    T = {}
    t0 = t()
    rs = b2.KlRankingSystem(pts, validate=False)
    tabs = rs.device_tables(); t1 = t(); T["tables(pin+h2d+prepare)"] = t1 - t0
    draws = b2.random_kout_draws(n, k, b2.derive_rng(0, 2)); t2 = t(); T["host draws"] = t2 - t1
    eng = Engine(n, k, tabs.device); table = eng.alloc_table(); eng.upload_rows(draws, table); t3 = t(); T["upload draws"] = t3 - t2
    R = cfg.resolved_max_rounds(n)
    smp = _to_device(draw_fcc_schedule(n, k, cfg, R), tabs.device); t4 = t(); T["fcc schedule"] = t4 - t3
    st, hist = descend_resident(eng, tabs, table, smp, 1000, R); t5 = t(); T["device descent"] = t5 - t4
    f = st.friends; t6 = t(); T["download+int64"] = t6 - t5
    T["total"] = t6 - t0
    print(rep, {k_: round(v * 1e3, 1) for k_, v in T.items()}, flush=True)
    t7 = t(); fr, h = b2.run(b2.Dataset(pts), b2.KlRankingSystem(pts, validate=False), cfg); print("  run()", round((t() - t7) * 1e3, 1), "ms")
