"""Golden fixtures (tests/golden/*.npz, produced from the UNMODIFIED reference by
tests/golden/make_golden.py) and the reference unit-test known answers
(proj/tests/unit/test_field.cpp) checked against the C restatement on the CPU, and against the
B200 library on the GPU (-m gpu).  These need neither /root/reference nor oracle/_ref, so they
also pin parity on the GPU box."""
import math
import os

import numpy as np
import pytest

import pyoracle as po

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name))


# ------------------------------------------------------------------ oracle vs golden (CPU)
@pytest.mark.parametrize("cfg", ["half", "cornell"])
def test_oracle_keys_golden(cfg):
    g = _load("keys.npz")
    o = po.OracleStore(po.Config.make(capacity_log2=8, base_cell_size=float(g[f"{cfg}_base"])))
    got = o.keys_for(g["pos"], g["dir"], g["level"])
    np.testing.assert_array_equal(np.ascontiguousarray(got).view(np.int32).reshape(-1, 7),
                                  g[f"{cfg}_keys"])


def test_oracle_levels_golden():
    g = _load("levels.npz")
    o = po.OracleStore(po.Config.make(capacity_log2=8, base_cell_size=float(g["base"]),
                                      max_level=int(g["max_level"])))
    np.testing.assert_array_equal(o.select_levels(g["footprint"]), g["level"])


def test_oracle_vertex_golden():
    g = _load("vertex.npz")
    kinds = (po.KIND_LO, po.KIND_LOE, po.KIND_FLI, po.KIND_LI)
    stores = [po.OracleStore(po.Config.make(kind=k, capacity_log2=int(g["cap"]),
                                            base_cell_size=float(g["base"]),
                                            evict_age_frames=int(g["evict"]))) for k in kinds]
    for it in range(int(g["frames"])):
        buf, n = po.synth_generate(int(g["width"]), int(g["height"]), int(g["bounces"]),
                                   iteration=it)
        po.vertex_pass_oracle(*stores, buf, n, deterministic=True)
        for si, s in enumerate(stores):
            s.end_frame()
            np.testing.assert_array_equal(np.frombuffer(s.slots().tobytes(), np.uint8),
                                          g[f"f{it}_s{si}_slots"])
            st = s.stats()
            np.testing.assert_array_equal(
                [st[x] for x in ("frame", "rejected", "dropped", "internal_errors", "live")],
                g[f"f{it}_s{si}_stats"])


# ------------------------------------------------------------------ reference unit-test KATs
def _small():
    return po.Config.make(capacity_log2=12, base_cell_size=0.5, max_level=4)  # test_field.cpp:19-25


def test_kat_key_golden_vector():
    """test_field.cpp:29-45"""
    s = po.OracleStore(_small())
    k = s.key_for((1.25, 2.5, -0.75), (0, 0, 1), 1)
    assert k.level == 1 and tuple(k.cell) == (1, 2, -1) and tuple(k.dir) == (2, 2)
    assert k.checksum != 0
    assert s.key_for((1.25, 2.5, -0.75), (0, 0, 1), 1).checksum == k.checksum


def test_kat_select_level():
    """test_field.cpp:58-70"""
    s = po.OracleStore(_small())
    assert s.select_level(0.5 / 4.0) == 0
    assert s.select_level(1e-9) == 0
    assert s.select_level(1e9) == 4
    l1, l2 = s.select_level(0.4), s.select_level(0.8)
    assert l2 == l1 + 1 and l1 >= 1 and l2 <= 3


def test_kat_blend_examples():
    """test_field.cpp:171-210 (alpha = 1, 0.5 and the 1/T floor)"""
    p, d = (0.1, 0.1, 0.1), (0, 0, 1)
    s = po.OracleStore(_small())
    k = s.key_for(p, d, 0)
    s.increment_counter(k, 8.0)
    s.accumulate(k, (7, 7, 7), 8.0)
    s.end_frame()
    assert abs(s.query_from_level(p, d, 0)[0][0] - 7.0) <= 7e-14
    s = po.OracleStore(_small())
    k = s.key_for(p, d, 0)
    s.increment_counter(k, 3000.0)
    s.accumulate(k, (1, 1, 1), 3000.0)
    s.end_frame()
    s.increment_counter(k, 1000.0)
    s.accumulate(k, (5, 5, 5), 1000.0)
    s.end_frame()
    assert abs(s.query_from_level(p, d, 0)[0][0] - 3.0) <= 3e-12
    s = po.OracleStore(_small())
    k = s.key_for(p, d, 0)
    s.increment_counter(k, 1e6)
    s.accumulate(k, (1, 1, 1), 1e6)
    s.end_frame()
    s.increment_counter(k, 1.0)
    s.accumulate(k, (65, 65, 65), 1.0)
    s.end_frame()
    expected = (1.0 - 1.0 / 64.0) * 1.0 + (1.0 / 64.0) * 65.0
    assert abs(s.query_from_level(p, d, 0)[0][0] - expected) <= 1e-12 * expected


def test_kat_counters_rejection_and_zero_weight():
    """test_field.cpp:72-124"""
    p, d = (0.1, 0.1, 0.1), (0, 0, 1)
    s = po.OracleStore(_small())
    k = s.key_for(p, d, 0)
    assert s.stats()["live"] == 0
    s.increment_counter(k, 0.0)
    assert s.stats()["live"] == 1
    s.end_frame()
    assert not s.query_from_level(p, d, 0)[1]
    s = po.OracleStore(_small())
    k = s.key_for(p, d, 0)
    s.increment_counter(k, 1.0)
    s.accumulate(k, (math.nan, 0, 0), 1.0)
    assert s.stats()["rejected"] == 1
    s.accumulate(k, (2, 2, 2), 1.0)
    s.end_frame()
    assert abs(s.query_from_level(p, d, 0)[0][0] - 2.0) <= 2e-12


def test_kat_query_fallback():
    """test_field.cpp:145-169"""
    s = po.OracleStore(_small())
    p, d = (0.3, 0.3, 0.3), (0, 0, 1)
    v, ok, fb, lv = s.query_from_level(p, d, 0)
    assert not ok and v == (0.0, 0.0, 0.0)
    k = s.key_for(p, d, 2)
    s.increment_counter(k, 1.0)
    s.accumulate(k, (1.5, 1.5, 1.5), 1.0)
    s.end_frame()
    v, ok, fb, lv = s.query_from_level(p, d, 2)
    assert ok and not fb and abs(v[0] - 1.5) < 1e-12
    v, ok, fb, lv = s.query_from_level(p, d, 1)
    assert ok and fb and lv == 2


# ------------------------------------------------------------------ B200 vs golden (GPU)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2005_07547_b200 as pb
    return torch, pb


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["half", "cornell"])
def test_gpu_keys_golden(cfg):
    torch, pb = _gpu()
    g = _load("keys.npz")
    s = pb.FieldStore(pb.FieldStoreConfig(capacity_log2=8, base_cell_size=float(g[f"{cfg}_base"])))
    got = s.key_for_batch(torch.from_numpy(g["pos"]), torch.from_numpy(g["dir"]),
                          torch.from_numpy(g["level"])).cpu().numpy()
    np.testing.assert_array_equal(got, g[f"{cfg}_keys"])


@pytest.mark.gpu
def test_gpu_levels_golden():
    torch, pb = _gpu()
    g = _load("levels.npz")
    s = pb.FieldStore(pb.FieldStoreConfig(capacity_log2=8, base_cell_size=float(g["base"]),
                                          max_level=int(g["max_level"])))
    got = s.select_level_batch(torch.from_numpy(g["footprint"])).cpu().numpy()
    np.testing.assert_array_equal(got, g["level"])


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["ordered", "atomic"])
def test_gpu_vertex_golden(mode):
    """The reference's deterministic replay, frame by frame: ORDERED bitwise in every slot field;
    ATOMIC bitwise in occupancy/keys/ages/c_old, values to 1e-9."""
    torch, pb = _gpu()
    import gpu_util as gu
    g = _load("vertex.npz")
    kinds = (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI, pb.KIND_LI)
    stores = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=int(g["cap"]),
                                                base_cell_size=float(g["base"]),
                                                evict_age_frames=int(g["evict"]))) for k in kinds]
    m = pb.MODE_ORDERED if mode == "ordered" else pb.MODE_ATOMIC
    for it in range(int(g["frames"])):
        buf, n = pb.synth_generate(int(g["width"]), int(g["height"]), int(g["bounces"]),
                                   iteration=it)
        pb.vertex_pass(*stores, buf, n, mode=m)
        pb.end_frame_all(stores)
        for si, s in enumerate(stores):
            ref = np.frombuffer(g[f"f{it}_s{si}_slots"].tobytes(), po.SLOT_DTYPE)
            got = s.slots()
            if mode == "ordered":
                gu.assert_slots_bitwise(got, ref)
            else:
                gu.assert_slots_close(got, ref, rtol=1e-9)
            st = s.stats()
            np.testing.assert_array_equal(
                [st[x] for x in ("frame", "rejected", "dropped", "internal_errors", "live")],
                g[f"f{it}_s{si}_stats"])
