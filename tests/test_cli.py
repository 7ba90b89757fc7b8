"""Command line (paper_2202_00517_b200.cli) against the reference's
(cli.py:93-208; its tests/test_cli.py): exit codes, stdout holding the report
alone, dataset files byte-identical to similarity.py:176-192's writers, and —
on the GPU — the reports of golden invocations recorded from the reference's
CLI (tests/golden/make_cli_golden.py), wall-clock fields removed."""

import base64
import csv
import io
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from cli_strip import strip_clock
from conftest import ROOT, load_json

import paper_2202_00517_b200 as b2
from paper_2202_00517_b200.cli import main


def run_cli(capsys, *argv):
    code = main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


@pytest.fixture(scope="module")
def golden():
    return load_json("cli_cases.json")


# ---- host-only behaviour (no device work happens before these exits) ----

def test_invalid_config_exits_2(capsys, caplog):
    code, out, err = run_cli(capsys, "run", "--n", "100", "--dim", "5", "--k", "100")
    assert code == 2 and out == "" and "need n > k >= 2" in caplog.text


def test_k_above_the_device_limit_exits_2(capsys, caplog):
    """K > 64 (the device join's limit; the reference has none) is a ConfigError
    with the reference CLI's exit code, raised before any device work."""
    code, out, err = run_cli(capsys, "run", "--n", "1000", "--dim", "5", "--k", "100")
    assert code == 2 and out == "" and "k must be <= 64" in caplog.text


def test_missing_size_flags_exit_2(capsys):
    assert run_cli(capsys, "run", "--k", "4")[0] == 2
    assert run_cli(capsys, "sweep", "--k", "4", "--dims", "3")[0] == 2


def test_oracle_guard_exits_2(capsys, caplog):
    code, out, err = run_cli(capsys, "run", "--n", "100001", "--dim", "2", "--k", "2", "--recall", "full")
    assert code == 2 and out == "" and "guard" in caplog.text


def test_witness_is_out_of_scope(capsys, caplog):
    code, out, err = run_cli(capsys, "witness", "--dim", "3", "--trials", "2")
    assert code == 2 and out == "" and "outside this build" in caplog.text


def test_argparse_rejects_bad_values(capsys):
    for argv in (["run", "--n", "0", "--dim", "3", "--k", "2"], ["run", "--n", "10", "--dim", "3", "--k", "2",
                                                                 "--workers", "x"],
                 ["sweep", "--n", "10", "--k", "2", "--dims", "3,-1"], ["run", "--k", "2", "--format", "xml"]):
        with pytest.raises(SystemExit) as e:
            main(argv)
        assert e.value.code == 2


def test_dataset_writers_match_reference_bytes(golden, tmp_path):
    pts = np.array(golden["points"])
    b2.save_points_csv(tmp_path / "p.csv", pts)
    b2.save_points_f64(tmp_path / "p.f64", pts)
    assert (tmp_path / "p.csv").read_text() == golden["csv_text"]
    assert (tmp_path / "p.f64").read_bytes() == base64.b64decode(golden["f64_b64"])
    for f in (b2.load_points_csv(tmp_path / "p.csv"), b2.load_points_f64(tmp_path / "p.f64")):
        assert f.dtype == np.float64 and np.array_equal(f, pts)


def test_dataset_reader_errors(tmp_path):
    (tmp_path / "h.f64").write_bytes(b"\x01\x00")
    with pytest.raises(ValueError, match="truncated header"):
        b2.load_points_f64(tmp_path / "h.f64")
    (tmp_path / "p.f64").write_bytes(np.array([3, 2], "<u4").tobytes() + b"\0" * 40)
    with pytest.raises(ValueError, match="expected 48 payload bytes"):
        b2.load_points_f64(tmp_path / "p.f64")


def test_bad_data_in_exits_2(capsys, tmp_path):
    code, out, err = run_cli(capsys, "run", "--k", "3", "--data-in", str(tmp_path / "missing.f64"))
    assert code == 2 and out == ""


# ---- device runs ----

@pytest.mark.gpu
def test_golden_invocations(golden, capsys, cuda):
    for case in golden["cases"]:
        code, out, _ = run_cli(capsys, *case["argv"])
        fmt = "csv" if "csv" in case["argv"] else "json"
        assert code == case["code"]
        assert strip_clock(out, fmt) == case["report"], case["argv"]


@pytest.mark.gpu
def test_out_file_and_workers(tmp_path, capsys, cuda):
    args = ["run", "--n", "250", "--dim", "4", "--k", "5", "--seed", "9", "--recall", "full"]
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    assert run_cli(capsys, *args, "--out", str(a))[:2] == (0, "")
    assert run_cli(capsys, *args, "--out", str(b), "--workers", "4")[0] == 0
    da, db = strip_clock(a.read_text(), "json"), strip_clock(b.read_text(), "json")
    assert da["spec"].pop("workers") == 1 and db["spec"].pop("workers") == 4
    assert da == db


@pytest.mark.gpu
def test_dataset_round_trip(tmp_path, capsys, cuda):
    common = ["--k", "5", "--seed", "4", "--recall", "full"]
    for name in ("points.f64", "points.csv"):
        path = tmp_path / name
        code, out1, _ = run_cli(capsys, "run", "--n", "200", "--dim", "4", *common, "--data-out", str(path))
        assert code == 0 and path.exists()
        code, out2, _ = run_cli(capsys, "run", "--data-in", str(path), *common)
        assert code == 0
        assert strip_clock(out1, "json") == strip_clock(out2, "json")


@pytest.mark.gpu
def test_module_entry_point(cuda):
    proc = subprocess.run([sys.executable, "-m", "paper_2202_00517_b200.cli", "run", "--n", "100", "--dim", "4",
                           "--k", "4", "--recall", "off"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                          env=dict(os.environ, PYTHONPATH=ROOT))
    assert proc.returncode == 0, proc.stderr
    assert json.loads(proc.stdout)["spec"]["n"] == 100
