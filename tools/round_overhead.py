"""Per-round host overhead of the engine: wall time of each round (host) against
the GPU time of its kernels (CUDA events around the round), at a size where the
GPU work is small.  usage: python tools/round_overhead.py [n d k]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_00517_b200 as b2  # noqa: E402
from paper_2202_00517_b200.descent import FccSchedule, descend_resident  # noqa: E402
from paper_2202_00517_b200.engine import Engine  # noqa: E402

n, d, k = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (20000, 20, 20)))
dev = torch.device("cuda", 0)
pts = b2.sample_simplex_uniform(d, n, b2.derive_rng(0, b2.STREAM_DATA, d))
rs = b2.KlRankingSystem(pts, validate=False)
tabs = rs.device_tables(dev)
cfg = b2.DescentConfig(k=k, seed=0)
R = cfg.resolved_max_rounds(n)
eng = Engine(n, k, dev)
draws = eng.alloc_table()
eng.upload_rows(b2.random_kout_draws(n, k, b2.derive_rng(0, 2)), draws)
smp = FccSchedule(n, k, cfg, R, dev)
for rep in range(4):
    table = draws.clone()
    marks = []
    ev0 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    t0 = time.perf_counter()

    def on_round(st, s):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((time.perf_counter(), e))

    state, hist = descend_resident(eng, tabs, table, smp, cfg.fcc_sample_count, R, on_round=on_round)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    gpu = ev0.elapsed_time(marks[-1][1])
    per = [(marks[i][0] - (marks[i - 1][0] if i else t0)) * 1e3 for i in range(len(marks))]
    print(f"rep {rep}: n={n} rounds {len(hist)} wall {wall:.3f} ms, round walls "
          f"{' '.join(f'{x:.3f}' for x in per)} ms", flush=True)

if os.environ.get("PROFILE"):
    import cProfile
    import pstats

    table = draws.clone()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        table = draws.clone()
        descend_resident(eng, tabs, table, smp, cfg.fcc_sample_count, R)
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)

if os.environ.get("TRACE"):
    from torch.profiler import ProfilerActivity, profile

    table = draws.clone()
    descend_resident(eng, tabs, table, smp, cfg.fcc_sample_count, R)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            table = draws.clone()
            descend_resident(eng, tabs, table, smp, cfg.fcc_sample_count, R)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    busy = sum(e.device_time for e in ev) / 1e3
    print(f"GPU kernel+copy time over 5 descents: {busy:.3f} ms ({len(ev)} device events)")
    print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25))
