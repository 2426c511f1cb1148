"""The reference's own field unit tests (proj/tests/unit/test_field.cpp, compiled in place from
/root/reference with a doctest shim, tests/native/Makefile):

* unit_field_ref  — against the unmodified reference field.cpp (CPU control; checks the shim and
                    the authored furnace scenes),
* unit_field_b200 — against the drop-in C++ facade over the B200 library (GPU).

Both binaries are built in this container by tests/native/Makefile (the reference tree does not
exist on the GPU box; the built binaries travel with the repo snapshot)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "native", "bin")

FIELD_CASES = [
    "key_for: quantization golden vector",
    "key_for: nearby positions share a key",
    "select_level: clamped log2 law",
    "counters and accumulation feed the density estimate",
    "compute_update_value: per-kind forms",
    "query: cold cache, read-back and coarse fallback",
    "end_frame: the three blending-coefficient examples",
    "end_frame: c_old stays capped",
    "temporal averaging: linear blend",
    "invalidate: global, regional, and the alpha reset",
    "density normalization",
    "jacobi discipline",
    "checksum safety",
    "eviction: overflowing inserts are dropped",
    "snapshot: dump and read round trip",
    "one-bounce field",
    "progressive convergence",
    "technique masks",
]


def _run(binary, case):
    exe = os.path.join(BIN, binary)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([exe, f"--tc={case}"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert "[PASS]" in r.stdout and "[FAIL]" not in r.stdout, r.stdout + r.stderr
    assert r.returncode == 0, r.stdout


@pytest.mark.parametrize("case", FIELD_CASES)
def test_reference_unit_tests_on_reference(case):
    _run("unit_field_ref", case)


@pytest.mark.gpu
@pytest.mark.parametrize("case", FIELD_CASES)
def test_reference_unit_tests_on_b200(case):
    _run("unit_field_b200", case)


@pytest.mark.gpu
def test_facade_load_snapshot_round_trip(tmp_path):
    """checkpoint/resume through the drop-in C++ facade: dumpSnapshot -> loadSnapshot (the
    facade's extension over pstf_field_load_snapshot) -> dumpSnapshot gives byte-identical files
    and identical queries; a snapshot of another field kind is refused (tests/native/
    facade_restore.cpp)."""
    exe = os.path.join(BIN, "facade_restore")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade restore ok" in r.stdout

