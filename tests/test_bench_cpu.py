"""bench.py's multi-rank launcher on CPU: ``--gpus 2`` outside torchrun must
re-launch itself with two ranks (torch.distributed.run, 127.0.0.1) and report
the whole group's result from rank 0 (gloo, ``--dry-run``)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*argv):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], env=env,
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_spawns_two_ranks():
    out = _run("--gpus", "2", "--steps", "2", "--warmup", "1", "--dry-run")
    assert out["n_gpus"] == 2 and out["ranks_seen"] == 2 and out["steps"] == 2


def test_bench_single_rank_dry_run():
    out = _run("--steps", "3", "--warmup", "1", "--dry-run")
    assert out["n_gpus"] == 1 and out["ranks_seen"] == 1
