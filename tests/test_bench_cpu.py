"""bench.py's launcher logic on CPU: `--gpus N` without WORLD_SIZE re-runs the command as N ranks
under torch.distributed.run (one process per GPU on a GPU box).  The reference arm needs no GPU:
rank 0 times the host path and prints the line, the other ranks exit 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TINY = ["--width", "48", "--height", "32", "--capacity-log2", "12", "--steps", "1", "--warmup",
        "1", "--streams", "2"]


def _run(args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_gpus_2_spawns_two_ranks():
    d = _run(TINY + ["--impl", "reference", "--gpus", "2"])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    if "unavailable" not in d:
        assert d["launched_ranks"] == 2  # WORLD_SIZE seen by rank 0 under the launcher
        assert d["config"]["parallelism"].startswith("2 ranks")


def test_single_rank_reference_line():
    d = _run(TINY + ["--impl", "reference"])
    assert d["n_gpus"] == 1 and d.get("launched_ranks", 1) == 1
