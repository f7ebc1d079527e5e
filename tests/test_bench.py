"""bench.py launch plumbing on CPU (no GPU): --gpus N spawns N ranks itself
(torch.distributed.run on 127.0.0.1, gloo in the dry run), seeds differ per
rank, timing is max over ranks and frames are summed over ranks; a
WORLD_SIZE that contradicts --gpus fails loudly."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=300, cwd=ROOT)


def test_gpus2_dry_run_spawns_two_ranks():
    p = _run(["--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "3", "--frames", "64"])
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert line["dry_run"] and line["n_gpus"] == 2
    assert line["frames_total"] == 2 * 64 * 2
    a, b = line["rank_first_llr"]
    assert a != b  # distinct frame seeds per rank


def test_gpus1_dry_run_single_process():
    p = _run(["--dry-run", "--steps", "1", "--frames", "16"])
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["frames_total"] == 16


def test_world_size_contradicting_gpus_fails_loudly():
    p = _run(["--gpus", "2", "--dry-run", "--steps", "1", "--frames", "16"], env={"WORLD_SIZE": "1"})
    assert p.returncode != 0
    assert "--gpus 2 but WORLD_SIZE=1" in p.stderr
