"""The reference's own acceptance criteria 4, 5, 9 and 10 (proj/tests/acceptance/
acceptance_main.cpp:202-239, 244-308, 475-504, 509-547), compiled in place from /root/reference
against the drop-in C++ facade over the B200 field cache (tests/native/bin/acceptance_b200) and,
as a control, against the reference field.cpp (acceptance_ref):
  4  progressive solver convergence on the furnaces (EstimatorRun PT_NEE, 2 workers, 256 frames)
  5  temporal averaging unit vectors (alpha = 1, 0.5, the 1/T floor, invalidate)
  9  density normalisation independent of sample density (256 frames x 10/100/1000 calls)
  10 deterministic mode bit-identical across runs and worker counts (CV estimator)
The GPU build must PASS every one; the binaries travel with the repo snapshot."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "native", "bin")
CRITERIA = (4, 5, 9, 10)


def _run(binary, criterion):
    exe = os.path.join(BIN, binary)
    if not os.path.exists(exe) or not os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "scenes")):
        pytest.skip(f"{exe} or oracle/_ref/scenes not built (needs /root/reference at build)")
    r = subprocess.run([exe, str(criterion)], cwd=ROOT, capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0 and "[PASS]" in r.stdout, r.stdout + r.stderr
    return r.stdout


@pytest.mark.parametrize("criterion", [5, 9, 10])
def test_acceptance_reference_control(criterion):
    _run("acceptance_ref", criterion)


@pytest.mark.gpu
@pytest.mark.parametrize("criterion", CRITERIA)
def test_acceptance_on_b200(criterion):
    print(_run("acceptance_b200", criterion))
