"""The run / sweep front end (cg/cli.py:42-228 flags and exit codes) on the
GPU path.  Configuration errors exit 1 before any device work, so those
cases run on CPU; the runs themselves are GPU tests."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2202_06111_b200", *args],
                          capture_output=True, text=True, timeout=600, cwd=cwd or str(ROOT))


@pytest.mark.parametrize("args,key", [
    (["run", "--model", "nope"], "model"),
    (["run", "--iterations", "0"], "iterations"),
    (["run", "--set", "linear.a"], "linear.a"),
    (["sweep", "--N", "1,x"], "N"),
])
def test_configuration_errors_exit_1(args, key, tmp_path):
    r = _cli(*args, "--output-dir", str(tmp_path / "out"))
    assert r.returncode == 1, r.stderr
    assert f"'{key}'" in r.stderr


@pytest.mark.gpu
def test_run_writes_outputs_and_empty_exits_3(tmp_path):
    r = _cli("run", "--model", "linear", "--iterations", "6", "--output-dir",
             str(tmp_path / "lin"), "--export-edges")
    assert r.returncode == 0, r.stderr
    for name in ("final.cells", "metrics.tsv", "timings.tsv", "summary.txt", "edges.tsv",
                 "effective.cfg"):
        assert (tmp_path / "lin" / name).exists(), name
    assert "termination = iterations" in (tmp_path / "lin" / "summary.txt").read_text()
    r = _cli("run", "--model", "shift", "--output-dir", str(tmp_path / "shift"))
    assert r.returncode == 3 and "no invariant set" in r.stderr


@pytest.mark.gpu
def test_sweep_over_N_and_plans(tmp_path):
    r = _cli("sweep", "--model", "cstr", "--iterations", "4", "--N", "0,3,full",
             "--workers", "1,2", "--output-dir", str(tmp_path / "sw"))
    assert r.returncode == 0, r.stderr
    rows = (tmp_path / "sw" / "sweep.tsv").read_text().splitlines()
    assert rows[0].startswith("point\titeration")
    points = {ln.split("\t")[0] for ln in rows[1:]}
    assert points == {f"N_{n}__workers_{w}" for n in ("0", "3", "full") for w in ("1", "2")}
    # BuildPlan.workers never changes a result: the metrics of w=1 and w=2 agree
    by = {}
    for ln in rows[1:]:
        p, rest = ln.split("\t", 1)
        by.setdefault(p.split("__")[0], set()).add((p.split("__")[1], rest))
    for n, entries in by.items():
        w1 = sorted(r for w, r in entries if w == "workers_1")
        w2 = sorted(r for w, r in entries if w == "workers_2")
        assert w1 == w2, n
