"""Reference outcomes for the behavioural API tests (build container only).

Runs the reference's run / run_to_fixed_point / init_random_kout on the small
instances its own test_descent.py uses (kl_instance / euclid_instance: points
from sample_simplex_uniform(d, n, seed), or standard normal vectors) and
records each result's sha256 and history, so tests/test_descent_api.py can
check the device engine against the reference on the same inputs.
Output: tests/golden/api_cases.json.
Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_api_golden.py
"""

import hashlib
import json
import os

import numpy as np
from rankdescent import (DescentConfig, Dataset, EuclideanRankingSystem, KlRankingSystem, derive_rng,
                         init_random_kout, run, run_to_fixed_point, sample_simplex_uniform)

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def kl(n, d, seed):
    pts = sample_simplex_uniform(d, n, seed)
    return Dataset(pts), KlRankingSystem(pts, validate=False)


def eu(n, d, seed):
    v = np.random.default_rng(seed).standard_normal((n, d))
    return Dataset(v), EuclideanRankingSystem(v)


def hist(h):
    return [[s.round_index, s.fcc, s.comparisons, s.changed_friend_sets] for s in h]


out = {}
for name, (mk, n, d, seed, kw) in {
    "run_kl_2000_6_k8_s20": (kl, 2000, 6, 20, dict(k=8, seed=20)),
    "run_kl_500_5_k6_s23": (kl, 500, 5, 23, dict(k=6, seed=23)),
    "run_kl_5_3_k4_s22": (kl, 5, 3, 22, dict(k=4, seed=22)),
    "run_kl_100_4_k4_s19_max1": (kl, 100, 4, 19, dict(k=4, seed=19, max_rounds=1)),
    "run_kl_30_4_k4_s21": (kl, 30, 4, 21, dict(k=4, seed=21)),
    "fixed_eu_120_3_k4_s25": (eu, 120, 3, 25, dict(k=4, seed=25)),
    "fixed_eu_120_3_k4_s26_max2": (eu, 120, 3, 26, dict(k=4, seed=26, max_rounds=2)),
}.items():
    ds, rs = mk(n, d, seed)
    fn = run_to_fixed_point if name.startswith("fixed") else run
    friends, h = fn(ds, rs, DescentConfig(**kw))
    out[name] = {"kind": mk.__name__, "n": n, "d": d, "seed": seed, "cfg": kw, "sha": sha(friends),
                 "history": hist(h)}
    print(name, len(h), flush=True)
for name, (n, d, seed, k, rseed) in {"init_kl_1000_5_k8_s42": (1000, 5, 42, 8, 42),
                                     "init_kl_300_6_k7_s3": (300, 6, 3, 7, 3),
                                     "init_kl_12_3_k6_s4": (12, 3, 4, 6, 4),
                                     "init_kl_5_3_k4_s1": (5, 3, 1, 4, 0)}.items():
    ds, rs = kl(n, d, seed)
    st = init_random_kout(ds, rs, DescentConfig(k=k), derive_rng(rseed, 2))
    out[name] = {"kind": "kl", "n": n, "d": d, "seed": seed, "k": k, "rng_seed": rseed, "sha": sha(st.friends)}
with open(os.path.join(HERE, "api_cases.json"), "w") as fh:
    json.dump(out, fh, indent=1)
