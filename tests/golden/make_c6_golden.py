"""The reference's acceptance C6 instances (test_acceptance.py: 50 Gaussian
point clouds run to a fixed point), recorded per instance: final-table sha256,
history length, recall against the reference's exact K-NN.
Output: tests/golden/c6_cases.json.
Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c6_golden.py
"""

import hashlib
import json
import os

import numpy as np
from rankdescent import DescentConfig, Dataset, EuclideanRankingSystem, exact_knn, recall, run_to_fixed_point

HERE = os.path.dirname(os.path.abspath(__file__))
gen = np.random.default_rng(606)
out = []
for i in range(50):
    n = int(gen.integers(20, 201))
    k = int(gen.choice([2, 4, 8]))
    d = int(gen.integers(2, 6))
    pts = gen.standard_normal((n, d))
    ds, rs = Dataset(pts), EuclideanRankingSystem(pts)
    friends, hist = run_to_fixed_point(ds, rs, DescentConfig(k=k, seed=i, max_rounds=1000))
    rec = recall(friends, exact_knn(ds, rs, k), np.arange(n))
    out.append({"i": i, "n": n, "k": k, "d": d, "rounds": len(hist), "recall": rec,
                "sha": hashlib.sha256(np.ascontiguousarray(friends, dtype=np.int32).tobytes()).hexdigest()})
print(sum(c["recall"] == 1.0 for c in out), "exact of 50")
with open(os.path.join(HERE, "c6_cases.json"), "w") as fh:
    json.dump(out, fh, indent=1)
