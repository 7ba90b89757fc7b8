"""Record the reference's own per-round trajectory for one configuration.

Runs ONLY in the build container (it imports the reference package from
/root/reference, which does not exist on the GPU box).  It drives the
reference's public functions exactly as ``rankdescent.run`` does
(descent.py:341-362: init_random_kout with derive_rng(seed, 2), then
run_round until the FCC stalls or max_rounds), and writes

  <out>/meta.json          per-round stats + sha256 of every round table
  <out>/table_rXX.npy      the int32 (n, K) table after round XX (00 = init)

The sha256 convention used everywhere in this repo is
``hashlib.sha256(np.ascontiguousarray(t, dtype='<i4').tobytes())``.

Usage: python tests/golden/record_reference.py --n 10000 --d 5 --k 10 --out /tmp/refruns/c1
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"


def table_sha(t: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(t, dtype="<i4").tobytes()).hexdigest()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--d", type=int, required=True)
    ap.add_argument("--k", type=int, required=True)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-rounds", type=int, default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--save-tables", type=int, default=1)
    args = ap.parse_args()

    sys.path.insert(0, REF_SRC)
    import rankdescent as rd  # noqa: E402  (reference, container-only)

    os.makedirs(args.out, exist_ok=True)
    spec = rd.ExperimentSpec(n=args.n, d=args.d, k=args.k, seed=args.seed, recall_mode="off")
    points = rd.bench.generate_points(spec)
    rs = rd.KlRankingSystem(points, validate=False)
    ds = rd.Dataset(points)
    cfg = rd.DescentConfig(k=args.k, seed=args.seed, max_rounds=args.max_rounds)
    max_rounds = cfg.resolved_max_rounds(args.n)

    meta = {
        "n": args.n, "d": args.d, "k": args.k, "seed": args.seed,
        "max_rounds": max_rounds,
        "points_sha": hashlib.sha256(np.ascontiguousarray(points, dtype="<f8").tobytes()).hexdigest(),
        "rounds": [],
    }
    t0 = time.perf_counter()
    state = rd.init_random_kout(ds, rs, cfg, rd.derive_rng(args.seed, 2))
    meta["init_sec"] = time.perf_counter() - t0
    meta["init_sha"] = table_sha(state.friends)
    if args.save_tables:
        np.save(os.path.join(args.out, "table_r00.npy"), state.friends.astype(np.int32))
    history = []
    for _ in range(max_rounds):
        state, st = rd.run_round(state, rs, cfg)
        history.append(st)
        rec = {
            "round": st.round_index, "sec": st.wall_clock_sec, "fcc": st.fcc,
            "fcc_count": int(round(st.fcc * cfg.fcc_sample_count)),
            "comparisons": int(st.comparisons), "changed": int(st.changed_friend_sets),
            "sha": table_sha(state.friends),
            "indeg_max": int(np.diff(state.cof_indptr).max()),
        }
        meta["rounds"].append(rec)
        print(json.dumps(rec), flush=True)
        if args.save_tables:
            np.save(os.path.join(args.out, f"table_r{st.round_index:02d}.npy"), state.friends.astype(np.int32))
        with open(os.path.join(args.out, "meta.json"), "w") as fh:
            json.dump(meta, fh, indent=1)
        if len(history) >= 2 and history[-1].fcc <= history[-2].fcc:
            break
    meta["total_sec"] = time.perf_counter() - t0
    meta["rounds_used"] = len(history)
    with open(os.path.join(args.out, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
