"""bench.py's multi-rank path on the GPU: `--gpus 2` re-launches itself as 2 ranks under
torch.distributed.run and rank 0 prints one JSON line with n_gpus 2.  With one GPU on the test
box the ranks share it and use gloo (PSTF_BENCH_BACKEND=gloo: collectives through the host, so
no kernel waits on another rank); the driver's multi-GPU runs use NCCL, one GPU per rank."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks(scaling):
    env = dict(os.environ, PSTF_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
                        "--width", "640", "--height", "360", "--scaling", scaling],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert "2 ranks" in line["config"]["parallelism"]
