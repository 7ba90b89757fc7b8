"""The stand-in for compute-sanitizer, which this GPU pool keeps closed
(tests/test_sanitize.py skips there): every libknnd kernel runs from the
bounds-checked build (libknnd_checked.so, -DKNND_CHECKED — device-side checks
on every hand-computed shared-memory, list, staging and workspace index) with
guard zones around every workspace (KNND_GUARD=1), over the sanitizer workload
(tools/sanitize_workload.py: init draws, row sort, CSR, every join size class
incl. the global-memory hub tables and the peer stores, K = 64, FCC,
batch_scores, the tensor-core exact K-NN, Euclidean), each result checked
against the C oracle.  Zero failed checks, zero guard bytes touched."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_and_guards_clean(cuda):
    lib = os.path.join(ROOT, "paper_2202_00517_b200", "libknnd_checked.so")
    assert os.path.exists(lib), "libknnd_checked.so missing: run __graft_entry__.build()"
    env = dict(os.environ, KNND_LIBRARY="checked", KNND_GUARD="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py")], capture_output=True,
                       text=True, timeout=1200, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "SANITIZE_OK" in out and "device bounds checks failed: 0 " in out and "guard bytes overwritten: 0" in out, \
        out[-4000:]
