"""bench.py launch plumbing on CPU: `bench.py --gpus N` run directly (as the
driver's BENCH step does) must spawn N ranks itself -- a scaling run can
never silently measure one GPU."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0]), r.stderr


def test_gpus_flag_spawns_ranks():
    line, err = _run("--gpus", "2", "--dry-run")
    assert line["n_gpus"] == 2 and line["ranks_reporting"] == 2
    assert "spawning 2 ranks" in err and "world 2" in err


def test_single_gpu_default_does_not_spawn():
    line, err = _run("--dry-run")
    assert line["n_gpus"] == 1 and "spawning" not in err
