"""bench.py's JSON-line contract (the driver parses it): a short run on the GPU at a reduced
frame prints one line with the required keys, a roofline and e2e object, clocks, kernel
launches, and the reference arm prints its own line.  Not a performance measurement."""
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
SMALL = ["--width", "320", "--height", "180", "--capacity-log2", "16", "--steps", "3",
         "--warmup", "3"]


def _line(args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_b200_line():
    d = _line(SMALL + ["--e2e-steps", "2", "--cpu-seconds", "2"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "gpu_launches", "roofline", "e2e", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["gpu_launches"] > 0 and "workload" in d["config"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.5
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-6
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["cpu_baseline"]["kind"] in ("reference", "port", "unavailable")


def test_reference_arm_line():
    d = _line(SMALL + ["--impl", "reference"])
    assert d.get("impl") == "reference"
    if "unavailable" in d:
        return
    assert d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"]


def test_sharded_branch_on_one_rank():
    """the multi-GPU branch (NCCL group, key-owner-sharded iteration with device-side exchange
    sizes, sharded e2e) run as a one-rank group: it must complete and print a valid line"""
    d = _line(SMALL + ["--force-sharded", "--no-cpu-baseline", "--e2e-steps", "2"])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "all-reduced" in d["config"]["parallelism"]



def test_reference_arm_config_matches_b200_arm():
    """both arms print the same `config` object for the same command line (the driver compares
    them), and the B200 line names its arm"""
    b = _line(SMALL + ["--no-e2e", "--no-cpu-baseline"])
    r = _line(SMALL + ["--impl", "reference"])
    assert b["impl"] == "b200" and r["impl"] == "reference"
    if "unavailable" not in r:
        assert b["config"] == r["config"]
