"""C ABI surface checks that need no GPU: the library loads, exports every function that
include/pstf_field.h declares, reports its ABI version, parses snapshot files, and refuses to
create a store without a CUDA device (there is no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "pstf_field.h")


@pytest.fixture(scope="module")
def lib():
    import paper_2005_07547_b200 as pb
    if not os.path.exists(pb.library_path()):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2005_07547_b200")],
                       check=True)
    return pb.lib()


def declared_functions():
    text = open(HDR).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pstf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_surface():
    fns = declared_functions()
    for must in ("pstf_field_create", "pstf_field_apply", "pstf_field_query",
                 "pstf_field_end_frame", "pstf_vertex_pass", "pstf_field_dump_snapshot"):
        assert must in fns


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (pstf_[a-z0-9_]+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    for f in declared_functions():
        assert getattr(lib, f) is not None


def test_abi_version(lib):
    assert lib.pstf_abi_version() == 2


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib._name], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_no_cpu_fallback_without_device(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import paper_2005_07547_b200 as pb
    with pytest.raises(pb.PstfError, match="no CUDA device"):
        pb.FieldStore(pb.FieldStoreConfig(capacity_log2=8))


def test_invalid_config_rejected(lib):
    import paper_2005_07547_b200 as pb
    with pytest.raises(pb.PstfError):
        pb.FieldStore(pb.FieldStoreConfig(capacity_log2=0))
    with pytest.raises(pb.PstfError):
        pb.FieldStore(pb.FieldStoreConfig(probe_window=0))


def test_read_snapshot_matches_reference_writer(tmp_path, lib):
    """pstf_read_snapshot parses files written by the reference dumpSnapshot (field.cpp:311-355)
    and rejects bad headers (test_field.cpp:426-434)."""
    import pyoracle as po
    import paper_2005_07547_b200 as pb
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    r = po.RefStore(po.Config.make(capacity_log2=10, base_cell_size=0.5))
    rng = np.random.default_rng(3)
    pos = rng.uniform(-4, 4, size=(300, 3))
    d = rng.normal(size=(300, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    for i in range(300):
        k = r.key_for(pos[i], d[i], i % 5)
        r.increment_counter(k, 1.0)
        r.accumulate(k, rng.uniform(0, 1, 3), 1.0)
    r.end_frame()
    path = str(tmp_path / "r.snap")
    r.dump_snapshot(path)
    kind, mine = pb.read_snapshot(path)
    kind2, theirs = po.read_snapshot(path)
    assert kind == kind2 == 0 and len(mine) == len(theirs) > 0
    for f in ("level", "cell", "dir", "checksum", "value", "c_old"):
        np.testing.assert_array_equal(mine[f], theirs[f])
    bad = tmp_path / "bad.snap"
    bad.write_bytes(b"NOTASNAP0000")
    with pytest.raises(pb.PstfError, match="not a field snapshot"):
        pb.read_snapshot(str(bad))


@pytest.mark.parametrize("kw", [dict(grid_resolution=0), dict(grid_resolution=300),
                                dict(kind=1, kd_leaf_count=48), dict(kind=1, kd_leaf_count=1),
                                dict(kind=1, kd_split_threshold=1.0),
                                dict(kind=2, gmm_components=0), dict(kind=2, gmm_components=9),
                                dict(kind=2, gmm_alpha_em=0.5), dict(kind=2, gmm_alpha_em=1.2),
                                dict(kind=3), dict(capacity_log2=0)])
def test_invalid_model_config_rejected(lib, kw):
    """the model store validates its configuration as the reference constructors do
    (models.cpp:17-18, 99-101, 203-204, 429-432) before touching the device"""
    import paper_2005_07547_b200 as pb
    with pytest.raises(pb.PstfError, match="must|kind"):
        pb.ModelStore(**kw)
