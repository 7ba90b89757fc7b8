"""compute-sanitizer memcheck over every libknnd kernel (tools/sanitize_workload.py:
init draws, row sort, CSR, every join size class incl. the global-memory hub
tables and the peer stores, K = 64, FCC, batch_scores, exact K-NN, Euclidean),
each result checked against the C oracle.  One sanitizer tool per process and
per GPU job: racecheck and synccheck run as separate jobs
(tools/gpu_sanitize.sh; logs in profiles/r02_sanitize_*.txt)."""

from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SANITIZER = "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SANITIZER), reason="compute-sanitizer not installed")
def test_memcheck_clean(cuda):
    cmd = [SANITIZER, "--tool", "memcheck", "--leak-check", "no", "--error-exitcode", "9", "--print-limit", "50",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    if r.returncode == 86 and "closed on this pool" in out:
        pytest.skip("compute-sanitizer is closed on this GPU pool (tests/test_checked.py is the stand-in)")
    assert r.returncode == 0, out[-4000:]
    assert "SANITIZE_OK" in out, out[-4000:]
    m = re.search(r"ERROR SUMMARY: (\d+) error", out)
    assert m and m.group(1) == "0", out[-4000:]
