"""Golden reports of the reference's experiment harness (build container only).

Runs the reference's bench.run_experiment / dimension_sweep (bench.py:136-192)
on small specs and records every deterministic field (per-round fcc,
comparisons, changed_friend_sets; rounds_used, round_budget, final_fcc,
recall).  It also re-serialises each report with the wall-clock fields
replaced by fixed values (round i -> 0.25*(i+1) s, total 1.5 s), so the
JSON / CSV emitters (bench.py:197-267) can be compared byte for byte.
Output: tests/golden/bench_reports.json.
Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bench_golden.py
"""

import dataclasses
import json
import os

from rankdescent import bench as rb

HERE = os.path.dirname(os.path.abspath(__file__))

SPECS = [
    dict(n=2000, d=5, k=10),
    dict(n=2000, d=5, k=10, recall_mode="full", output_format="csv"),
    dict(n=1500, d=8, k=12, seed=3, max_rounds=3),
    dict(n=3000, d=3, k=8, ranking="euclidean"),
    dict(n=1200, d=4, k=6, seed=1, fcc_samples=300, recall_mode="off", output_format="csv"),
]
SWEEP = (dict(n=1500, k=6, d=2, seed=2), [3, 6])


def fixed_clock(rep):
    rounds = [dataclasses.replace(r, wall_clock_sec=0.25 * (i + 1)) for i, r in enumerate(rep.rounds)]
    return dataclasses.replace(rep, rounds=rounds, total_duration_sec=1.5)


def record(rep):
    return {
        "spec": rep.spec.to_dict(),
        "rounds": [[r.round_index, r.fcc, r.comparisons, r.changed_friend_sets] for r in rep.rounds],
        "rounds_used": rep.rounds_used,
        "round_budget": rep.round_budget,
        "final_fcc": rep.final_fcc,
        "recall": rep.recall,
        "emit_json": rb.emit_report(fixed_clock(rep), "json"),
        "emit_csv": rb.emit_report(fixed_clock(rep), "csv"),
    }


out = {"reports": [], "sweep": None}
for s in SPECS:
    rep = rb.run_experiment(rb.ExperimentSpec(**s))
    out["reports"].append(record(rep))
    print(s, rep.rounds_used, rep.recall, flush=True)
base, dims = SWEEP
reps = rb.dimension_sweep(rb.ExperimentSpec(**base), dims)
fixed = [fixed_clock(r) for r in reps]
out["sweep"] = {"base": base, "dims": dims, "reports": [record(r) for r in reps],
                "emit_json": rb.emit_sweep(fixed, "json"), "emit_csv": rb.emit_sweep(fixed, "csv")}
with open(os.path.join(HERE, "bench_reports.json"), "w") as fh:
    json.dump(out, fh, indent=1)
