"""bench.py's multi-rank launcher on CPU: `--gpus 2`
started as a plain process re-executes itself under torch.distributed.run
with two ranks; the dry-run arm inits gloo, reduces the step time as the max
over ranks, and rank 0 alone prints one JSON line with n_gpus == 2."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(*extra, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *extra], capture_output=True,
                          text=True, timeout=300, env=e, cwd=str(ROOT))


def _lines(out):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_launcher_spawns_two_ranks_and_rank0_prints_one_line():
    r = _run("--gpus", "2", "--steps", "3", "--warmup", "1", "--dry-run")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1, r.stdout
    ln = lines[0]
    assert ln["n_gpus"] == 2 and ln["steps"] == 3 and ln["warmup"] == 1
    assert ln["config"]["local_rank_env"] == "0"
    assert ln["value"] > 0 and ln["ms_per_step"] > 0


def test_single_rank_dry_run():
    r = _run("--steps", "2", "--warmup", "1", "--dry-run")
    assert r.returncode == 0, r.stderr[-2000:]
    (ln,) = _lines(r.stdout)
    assert ln["n_gpus"] == 1


def test_launcher_refuses_more_gpus_than_visible():
    r = _run("--gpus", "4", "--steps", "1", "--warmup", "1",
             env={"CUDA_VISIBLE_DEVICES": ""})
    assert r.returncode == 2
    assert "GPU(s) visible" in r.stderr
    assert _lines(r.stdout) == []
