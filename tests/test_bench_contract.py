"""bench.py's driver contract, the parts that run without a GPU: the
reference arm's JSON line (rank 0 only, bounded CPU sample through the C
oracle) and the B200 arm failing loudly — no CPU fallback — when no device
is present."""

import json
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config")


def _bench(*argv, env=None):
    return subprocess.run([sys.executable, "bench.py", *argv], cwd=ROOT, capture_output=True, text=True,
                          timeout=300, env=dict(os.environ, **(env or {})))


def test_reference_arm_line():
    p = _bench("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1", "--no-python-reference")
    assert p.returncode == 0, p.stderr
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and all(k in d for k in KEYS)
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0 and d["unit"] == "comparisons/s"
    assert d["higher_is_better"] is True and d["config"]["workload"].startswith("C1")
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # a step is the full descent (like the B200 arm's): the reference's own C1 trajectory
    with open(os.path.join(ROOT, "tests", "golden", "trajectories.json")) as fh:
        ref = json.load(fh)["c1"]
    assert d["config"]["rounds_per_step"] == [ref["rounds_used"]] * 2
    assert d["config"]["comparisons_per_step"] == sum(r["comparisons"] for r in ref["rounds"])
    assert d["config"]["final_table_sha256"] == ref["rounds"][-1]["sha"]


def test_reference_arm_other_ranks_are_silent():
    p = _bench("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0", env={"RANK": "1"})
    assert p.returncode == 0 and p.stdout.strip() == ""


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device failure")
def test_b200_arm_fails_loudly_without_a_device():
    p = _bench("--config", "c1", "--steps", "1", "--warmup", "3")
    assert p.returncode != 0
    assert not any(l.startswith("{") for l in p.stdout.splitlines())
