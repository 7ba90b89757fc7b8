"""Generate the golden fixtures in tests/golden/ from the reference itself.

Runs ONLY in the build container: it imports the reference package from
/root/reference/pkg/src (read-only, never copied into this repo).  The GPU
box never runs this; it reads the committed outputs:

  small_cases.npz      per case: init table, round-1 table, final table
  small_cases.json     per case: points sha, per-round stats and table
                       sha256 of a full run()
  trajectories.json    per-round stats + table sha256 of the BASELINE
                       configs, recorded by record_reference.py
                       (C1 n=10k d=5 K=10; C2 n=100k d=10 K=20; C3 n=1M d=20 K=20)
  known_answers.json   hand KL values from the reference's tests
                       (t_similarity:32-37, t_core:38-49), FCC extremes
                       (t_descent:286-294), round_budget pairs (t_descent:44-62)

Usage: python tests/golden/make_golden.py [--trajectories /tmp/refruns]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"

# (name, n, d, K, seed): covers both init regimes (rejection / dense
# permutation), K <= 32 and K > 32, the templated row widths d = 5/10/20/50
# and the generic one (d = 16), and the forced complete case.
SMALL_CASES = [
    ("n300_d6_k7_s3", 300, 6, 7, 3),
    ("n500_d5_k6_s23", 500, 5, 6, 23),
    ("n2000_d6_k8_s20", 2000, 6, 8, 20),
    ("n1000_d20_k20_s1", 1000, 20, 20, 1),
    ("n1500_d16_k10_s7", 1500, 16, 10, 7),
    ("n600_d50_k30_s2", 600, 50, 30, 2),
    ("n800_d10_k40_s5", 800, 10, 40, 5),
    ("n5_d3_k4_s22", 5, 3, 4, 22),
    ("n12_d3_k6_s4", 12, 3, 6, 4),
    ("n4000_d5_k10_s0", 4000, 5, 10, 0),
]


def sha_i32(t) -> str:
    return hashlib.sha256(np.ascontiguousarray(t, dtype="<i4").tobytes()).hexdigest()


def sha_f64(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def small_cases(rd) -> dict:
    out = {}
    meta = {}
    for name, n, d, k, seed in SMALL_CASES:
        spec = rd.ExperimentSpec(n=n, d=d, k=k, seed=seed, recall_mode="off")
        pts = rd.bench.generate_points(spec)
        rs = rd.KlRankingSystem(pts, validate=False)
        cfg = rd.DescentConfig(k=k, seed=seed)
        state = rd.init_random_kout(rd.Dataset(pts), rs, cfg, rd.derive_rng(seed, 2))
        out[f"{name}/init"] = state.friends.astype(np.int32)
        rounds = []
        hist = []
        for _ in range(cfg.resolved_max_rounds(n)):
            state, st = rd.run_round(state, rs, cfg)
            hist.append(st)
            if st.round_index == 1:
                out[f"{name}/round1"] = state.friends.astype(np.int32)
            rounds.append({"round": st.round_index, "comparisons": int(st.comparisons),
                           "changed": int(st.changed_friend_sets), "fcc": st.fcc,
                           "fcc_count": int(round(st.fcc * cfg.fcc_sample_count)), "sha": sha_i32(state.friends)})
            if len(hist) >= 2 and hist[-1].fcc <= hist[-2].fcc:
                break
        # the same run through the public entry point must agree
        final, h2 = rd.run(rd.Dataset(pts), rs, cfg)
        assert sha_i32(final) == rounds[-1]["sha"] and len(h2) == len(rounds)
        out[f"{name}/final"] = final.astype(np.int32)
        meta[name] = {"n": n, "d": d, "k": k, "seed": seed, "points_sha": sha_f64(pts),
                      "init_sha": sha_i32(out[f"{name}/init"]), "rounds": rounds}
        print(name, len(rounds), "rounds", flush=True)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **out)
    with open(os.path.join(HERE, "small_cases.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    return meta


def known_answers(rd) -> dict:
    pts = np.array([[0.5, 0.5], [0.25, 0.75], [0.1, 0.9]])
    rs = rd.KlRankingSystem(pts)
    ka = {
        "kl_points": pts.tolist(),
        "kl_01": rs.score(0, 1), "kl_02": rs.score(0, 2), "kl_10": rs.score(1, 0),
        "round_budget": [[n, k, rd.round_budget(n, k)] for n, k in
                         [(20000, 16), (20000, 32), (200000, 16), (200000, 32), (2000000, 16), (2000000, 32),
                          (2000000, 64), (256, 16), (16, 16), (10000, 10), (100000, 20), (1000000, 20),
                          (1000000, 30), (10000000, 20)]],
        "fcc_complete": rd.friend_clustering_rate(rd.KnnState(np.array([[1, 2], [0, 2], [0, 1]])), 500,
                                                  rd.derive_rng(0, 3, 1)),
        "fcc_bipartite": rd.friend_clustering_rate(rd.KnnState(np.array([[2, 3], [2, 3], [0, 1], [0, 1]])), 500,
                                                   rd.derive_rng(1, 3, 1)),
    }
    # batch_scores of a seeded simplex set against a few anchors (value pins)
    p2 = rd.sample_simplex_uniform(10, 300, 8)
    r2 = rd.KlRankingSystem(p2)
    ka["batch_points_sha"] = sha_f64(p2)
    ka["batch_scores"] = {str(x): r2.batch_scores(x).tolist() for x in (0, 3, 299)}
    with open(os.path.join(HERE, "known_answers.json"), "w") as fh:
        json.dump(ka, fh, indent=1)
    return ka


def trajectories(src: str) -> None:
    out = {}
    for name in ("c1", "c2", "c3", "c4"):
        p = os.path.join(src, name, "meta.json")
        if os.path.exists(p):
            with open(p) as fh:
                out[name] = json.load(fh)
    with open(os.path.join(HERE, "trajectories.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("trajectories:", {k: len(v["rounds"]) for k, v in out.items()})


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--trajectories", default=None, help="directory of record_reference.py outputs")
    ap.add_argument("--skip-small", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, REF_SRC)
    import rankdescent as rd  # reference, container-only

    if not args.skip_small:
        small_cases(rd)
        known_answers(rd)
    if args.trajectories:
        trajectories(args.trajectories)


if __name__ == "__main__":
    main()
