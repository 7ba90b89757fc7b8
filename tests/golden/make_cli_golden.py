"""Golden outputs of the reference's command line (build container only).

Runs the reference's ``rankdescent.cli.main`` (cli.py:196-208) on small
``run`` / ``sweep`` invocations and records the reports with the wall-clock
fields removed (JSON: rounds[].wall_clock_sec and the summary's
total/first/last seconds; CSV: those columns), plus the bytes of the
reference's dataset writers (similarity.py:176-192) for one small point set.
Output: tests/golden/cli_cases.json.
Usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py
"""

import base64
import contextlib
import io
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from cli_strip import strip_clock  # noqa: E402

from rankdescent import cli  # noqa: E402
from rankdescent.similarity import sample_simplex_uniform, save_points_csv, save_points_f64  # noqa: E402
from rankdescent.descent import derive_rng  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    ["run", "--n", "300", "--dim", "5", "--k", "6", "--seed", "3", "--recall", "full"],
    ["run", "--n", "200", "--dim", "4", "--k", "4", "--recall", "off", "--format", "csv"],
    ["run", "--n", "250", "--dim", "4", "--k", "5", "--seed", "9", "--ranking", "euclidean", "--max-rounds", "3"],
    ["sweep", "--n", "200", "--k", "4", "--dims", "4,6", "--recall", "full", "--format", "csv"],
    ["sweep", "--n", "150", "--k", "4", "--dims", "5", "--recall", "off"],
]


def main():
    out = {"cases": []}
    for argv in CASES:
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            code = cli.main(list(argv))
        fmt = "csv" if "csv" in argv else "json"
        out["cases"].append({"argv": argv, "code": code, "report": strip_clock(buf.getvalue(), fmt)})
    pts = sample_simplex_uniform(3, 5, derive_rng(7, 1, 3))
    with tempfile.TemporaryDirectory() as td:
        save_points_csv(os.path.join(td, "p.csv"), pts)
        save_points_f64(os.path.join(td, "p.f64"), pts)
        out["points"] = pts.tolist()
        out["csv_text"] = open(os.path.join(td, "p.csv")).read()
        out["f64_b64"] = base64.b64encode(open(os.path.join(td, "p.f64"), "rb").read()).decode()
    with open(os.path.join(HERE, "cli_cases.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
