"""Recall@K of the reference's final tables (build container only).

Exact neighbours of the reference's recall sample (evaluation.py:135-137,
uniform_recall_sample(n, seed, size)) are computed with the C oracle's brute
force (pinned to the reference's exact_knn loop body in tests/test_oracle.py),
and recall (evaluation.py:111-132) of the recorded final table is stored in
tests/golden/recall.json, for the full sample and for its first 2000 ids.
Usage: python tests/golden/make_recall.py /tmp/refruns [c1 c2 c3 c4 c5]
(configs not named keep their stored values; C5 was recorded separately,
its n = 10M brute force takes a while on the build container's cores)
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import native, port  # noqa: E402

src = sys.argv[1]
names = sys.argv[2:] or ["c1", "c2", "c3", "c4"]
path = os.path.join(HERE, "recall.json")
out = json.load(open(path)) if os.path.exists(path) else {}
for name, size in (("c1", None), ("c2", 10_000), ("c3", 10_000), ("c4", 10_000), ("c5", 10_000)):
    if name not in names:
        continue
    meta = json.load(open(os.path.join(src, name, "meta.json")))
    n, d, k, seed = meta["n"], meta["d"], meta["k"], meta["seed"]
    final = np.load(os.path.join(src, name, f"table_r{meta['rounds_used']:02d}.npy"))
    tab = native.Tables(port.experiment_points(n, d, seed))
    q = np.arange(n) if size is None else port.recall_sample(n, seed, size)
    exact = native.exact_rows(tab, q, k)
    rec = port.recall_of(final, exact, q)
    rec2k = port.recall_of(final, exact[:2000], q[:2000])
    out[name] = {"sample": "all" if size is None else f"uniform_recall_sample(n, {seed}, {size})",
                 "recall": rec, "recall_first2000": rec2k}
    print(name, out[name], flush=True)
with open(path, "w") as fh:
    json.dump(out, fh, indent=1)
