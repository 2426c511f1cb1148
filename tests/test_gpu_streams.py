"""Fused vertex-pass parity on real and adversarial streams (the fused kernels against the
reference itself, not against the synthetic generator's closed-box stream only).

1. Captured streams: the UNMODIFIED reference path tracer (oracle/_ref/libpstf_capture.so,
   pathtracer.cpp:80-239) renders a reference scene with a PathHooks collector
   (test_pathtracer.cpp:14-17); every frame's VertexRecords become the canonical SoA record and
   go through pstf_vertex_pass.  The ground truth is the reference's own EstimatorRun
   (estimators.cpp:308-655, PT_NEE, deterministic) rendering the same frames with its own
   field stores:
     * ORDERED mode: every slot (occupancy, key fields, valueOld, cOld, accumulators, ages) and
       the snapshot files are byte-identical, every frame;
     * ATOMIC mode through the TMA-tiled fused kernel: occupancy, key fields, ages and cOld
       bitwise, valueOld within rtol 1e-9 (per-vertex aggregation reassociates fp64 sums);
   Config 1 (BASELINE configs[0]) is cornell.scene at 256x256, 32 frames, capacity 2^18.
   Glossy (staircase_glossy.scene) and environment-lit (furnace_env.scene: escapes,
   estimators.cpp:207-210) scenes, technique masks other than 7 and the Li store as well.
2. Crafted streams (tests/crafted.py): escapes, NaN/inf/negative values, ratio <= 0, all flag
   combinations, boundary-hugging and non-finite positions/directions/footprints, tails that are
   not a multiple of the tile, masks 1..7; against the reference replay of onVertex
   (oracle/ref_shim.cpp, bitwise-pinned to EstimatorRun by tests/test_capture_pin.py).
3. One full config-2 iteration pair (1920x1080x4, 8,294,400 vertices, 2^22 slots) through the
   tiled kernel against the reference replay."""
import numpy as np
import pytest

import crafted
import gpu_util as gu
import pyoracle as po

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2005_07547_b200 as pb  # noqa: E402

try:
    import pycapture as pc
except Exception:  # pragma: no cover
    pc = None

KINDS = (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI, pb.KIND_LI)
WHICH = {pb.KIND_LO: 0, pb.KIND_LO_MINUS_E: 1, pb.KIND_FLI: 2, pb.KIND_LI: 3}


def _need_capture():
    if pc is None or not pc.available():
        pytest.skip("oracle/_ref/libpstf_capture.so not built (needs /root/reference at build)")


def _gpu_stores(cfg, li, masks=(7, 7)):
    kinds = KINDS if li else KINDS[:3]
    out = []
    for k in kinds:
        m = masks[0] if k == pb.KIND_LO_MINUS_E else (masks[1] if k == pb.KIND_FLI else 7)
        out.append(pb.FieldStore(pb.FieldStoreConfig(
            kind=k, capacity_log2=cfg["capacity_log2"], max_level=cfg["max_level"],
            base_cell_size=cfg["base_cell_size"], level_select_k=cfg["level_select_k"],
            t_max=cfg["t_max"], technique_mask=m, probe_window=cfg["probe_window"],
            evict_age_frames=cfg["evict_age_frames"])))
    return out


def _pass(st, dev, soa, n, masks, mode):
    li = st[3] if len(st) > 3 else None
    pb.vertex_pass(st[0], st[1], st[2], li, dev, n, loe_mask=masks[0], fli_mask=masks[1],
                   mode=mode, soa=soa)
    pb.end_frame_all(st)


def _ref_stats_equal(g, stats):
    s = g.stats()
    for k in ("frame", "rejected", "dropped", "internal_errors", "live"):
        assert s[k] == stats[k], (k, s[k], stats[k])


def _run_captured(scene_name, size, frames, li=False, masks=(7, 7), cap_log2=18, tmp=None,
                  snap_every=8):
    _need_capture()
    sc = pc.Scene(scene_name, size, size)
    run = pc.RefEstimatorRun(sc, kind=pc.PT_NEE, deterministic=True, capacity_log2=cap_log2,
                             track_li=li, loe_mask=masks[0], fli_mask=masks[1])
    cfg = run.store_config(0)
    ordered = _gpu_stores(cfg, li, masks)
    atomic = _gpu_stores(cfg, li, masks)
    seen = {"escape": 0, "ratio_le0": 0, "n": 0}
    pb.profile_enable(True)
    pb.profile_collect()
    try:
        for f in range(frames):
            buf, n = pc.capture_frame(sc, f, seed=0)
            fl = buf[34 * n:].view(np.uint32)[:n]
            ratio = buf[17 * n:18 * n]
            seen["escape"] += int(((fl & 1) != 0).sum() - ((fl & 3) == 3).sum())
            seen["ratio_le0"] += int((((fl & 1) != 0) & ~(ratio > 0)).sum())
            seen["n"] += n
            dev, soa = gu.device_stream(buf, n, pad=True)
            _pass(ordered, dev, soa, n, masks, pb.MODE_ORDERED)
            _pass(atomic, dev, soa, n, masks, pb.MODE_ATOMIC)
            assert gu.launched("k_vertex_pass_tiled"), "ATOMIC pass did not use the tiled kernel"
            run.frame()
            for w, (go, ga) in enumerate(zip(ordered, atomic)):
                ref = run.slots(w)
                gu.assert_slots_bitwise(go.slots(), ref)
                gu.assert_slots_close(ga.slots(), ref, rtol=1e-9, atol=1e-300)
                st = run.stats(w)
                _ref_stats_equal(go, st)
                _ref_stats_equal(ga, st)
            if tmp is not None and (f % snap_every == snap_every - 1 or f == frames - 1):
                for w, go in enumerate(ordered):
                    a, b = tmp / f"ref{w}.snap", tmp / f"gpu{w}.snap"
                    run.dump_snapshot(w, a)
                    go.dumpSnapshot(str(b))
                    assert a.read_bytes() == b.read_bytes(), (f, w)
    finally:
        pb.profile_enable(False)
    return seen


def test_captured_cornell_config1(tmp_path):
    """BASELINE configs[0]: cornell.scene 256x256, 1 spp, 32 frames, EstimatorRun defaults
    (capacity 2^18, base = diameter/256) — the reference CPU run, replayed on the B200 cache."""
    seen = _run_captured("cornell.scene", 256, 32, tmp=tmp_path)
    assert seen["n"] > 32 * 150_000


@pytest.mark.parametrize("scene,size,frames,li,masks", [
    ("staircase_glossy.scene", 128, 8, False, (7, 7)),
    ("staircase_glossy.scene", 96, 6, True, (2, 4)),
    ("furnace_env.scene", 64, 6, False, (7, 7)),
    ("furnace_env.scene", 64, 4, True, (4, 2)),
    ("cornell.scene", 96, 5, True, (6, 3)),
    ("cornell_door.scene", 96, 5, False, (1, 5)),
])
def test_captured_scenes(tmp_path, scene, size, frames, li, masks):
    seen = _run_captured(scene, size, frames, li=li, masks=masks, tmp=tmp_path, snap_every=4)
    if scene == "furnace_env.scene":
        assert seen["escape"] > 0, "environment escapes expected"


# ------------------------------------------------------------------------ crafted streams
def _ref_stores(cfg_kw, li, masks):
    kinds = (po.KIND_LO, po.KIND_LOE, po.KIND_FLI) + ((po.KIND_LI,) if li else ())
    out = []
    for k in kinds:
        m = masks[0] if k == po.KIND_LOE else (masks[1] if k == po.KIND_FLI else 7)
        c = po.Config.make(kind=k, technique_mask=m, **cfg_kw)
        out.append(po.RefStore(c) if po.ref_available() else po.OracleStore(c))
    return out


@pytest.mark.parametrize("li", [False, True])
@pytest.mark.parametrize("pad", [True, False])
def test_crafted_streams(li, pad):
    """adversarial streams through ATOMIC (tiled kernel when pad=True, the per-thread kernel on
    unaligned fields when pad=False) and ORDERED, frame after frame with changing masks"""
    base = (12.0 ** 0.5) / 256.0
    cfg_kw = dict(capacity_log2=15, base_cell_size=base)
    gcfg = dict(capacity_log2=15, max_level=4, base_cell_size=base, level_select_k=4.0,
                t_max=64.0, probe_window=32, evict_age_frames=64)
    g_ord, g_atm = _gpu_stores(gcfg, li), _gpu_stores(gcfg, li)
    r_ord, r_atm = _ref_stores(cfg_kw, li, (7, 7)), _ref_stores(cfg_kw, li, (7, 7))
    for f in range(7):
        masks = (1 + f % 7, 1 + (3 * f + 1) % 7)
        buf0, n0 = po.synth_generate(96, 54, 4, iteration=f)
        n = n0 - 37 - 2 * f  # a tail that is not a multiple of the 128-vertex tile
        f64, fl = crafted.views(buf0, n0)
        buf = np.zeros(34 * n + (n + 1) // 2)
        fo, flo = crafted.views(buf, n)
        fo[:] = f64[:, :n]
        flo[:] = fl[:n]
        ext = crafted.mutate(buf.copy(), n, seed=1000 + f, base=base, extreme=True)
        mod = crafted.mutate(buf.copy(), n, seed=2000 + f, base=base, extreme=False)
        # per-frame masks: the stores' technique_mask is carried but not read (field.h:54);
        # the pass takes the masks (estimators.cpp:228-250)
        lr = r_ord[3] if li else None
        po.vertex_pass_ref(r_ord[0], r_ord[1], r_ord[2], lr, ext, n, masks[0], masks[1],
                           deterministic=True)
        la = r_atm[3] if li else None
        po.vertex_pass_ref(r_atm[0], r_atm[1], r_atm[2], la, mod, n, masks[0], masks[1],
                           deterministic=True)
        for s in r_ord + r_atm:
            s.end_frame()
        dev, soa = gu.device_stream(ext, n, pad=pad)
        _pass(g_ord, dev, soa, n, masks, pb.MODE_ORDERED)
        dev, soa = gu.device_stream(mod, n, pad=pad)
        pb.profile_enable(True)
        pb.profile_collect()
        _pass(g_atm, dev, soa, n, masks, pb.MODE_ATOMIC)
        tiled = gu.launched("k_vertex_pass_tiled")
        pb.profile_enable(False)
        assert bool(tiled) == pad
        for go, ga, ro, ra in zip(g_ord, g_atm, r_ord, r_atm):
            gu.assert_slots_bitwise(go.slots(), ro.slots())
            gu.assert_slots_close(ga.slots(), ra.slots(), rtol=1e-9, atol=1e-12)
            _ref_stats_equal(go, ro.stats())
            _ref_stats_equal(ga, ra.stats())
    assert sum(s.stats()["rejected"] for s in r_atm) > 0


# --------------------------------------------------- config 3: glossy stream + CV at every vertex
def test_glossy_stream_with_cv_lookup():
    """BASELINE config 3 shape at a reduced frame: the glossy synthetic stream (scene 1) through
    the tiled kernel with the fused CV lookup (estimators.cpp:453-462) against the reference
    replay; the CV outputs equal the reference's LoE query on the frame-start table"""
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    base = (12.0 ** 0.5) / 256.0
    gcfg = dict(capacity_log2=16, max_level=4, base_cell_size=base, level_select_k=4.0,
                t_max=64.0, probe_window=32, evict_age_frames=64)
    g = _gpu_stores(gcfg, False)
    r = _ref_stores(dict(capacity_log2=16, base_cell_size=base), False, (7, 7))
    for it in range(5):
        host, n = po.synth_generate(192, 108, 4, iteration=it, scene=1)
        dev, soa = gu.device_stream(host, n, pad=True)
        f64, _ = crafted.views(host, n)
        want_v, want_ok, _, _ = r[1].query_batch(f64[0:3].T, f64[3:6].T, fp=f64[15])
        pb.profile_enable(True)
        pb.profile_collect()
        val, ok = pb.vertex_pass_cv(g[0], g[1], g[2], None, dev, n, soa=soa)
        assert gu.launched("k_vertex_pass_tiled")
        pb.profile_enable(False)
        pb.end_frame_all(g)
        po.vertex_pass_ref(r[0], r[1], r[2], None, host, n, deterministic=True)
        for s in r:
            s.end_frame()
        np.testing.assert_array_equal(ok.cpu().numpy().astype(bool), np.asarray(want_ok, bool))
        np.testing.assert_allclose(val.cpu().numpy().T, want_v, rtol=1e-9, atol=1e-300)
        for a, b in zip(g, r):
            gu.assert_slots_close(a.slots(), b.slots(), rtol=1e-9, atol=1e-300)
            _ref_stats_equal(a, b.stats())


# ------------------------------------------------------------- one full config-2 iteration
@pytest.mark.slow
def test_config2_full_iterations_vs_reference():
    """BASELINE configs[1] at full size: two 8,294,400-vertex iterations (the first inserts
    every key, the second is the steady state of existing-slot REDs) through the tiled ATOMIC
    kernel against the reference's deterministic replay: keys, occupancy, ages and cOld
    bitwise, values within 1e-9."""
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    base = (12.0 ** 0.5) / 256.0
    gcfg = dict(capacity_log2=22, max_level=4, base_cell_size=base, level_select_k=4.0,
                t_max=64.0, probe_window=32, evict_age_frames=64)
    g = _gpu_stores(gcfg, False)
    r = _ref_stores(dict(capacity_log2=22, base_cell_size=base), False, (7, 7))
    threads = 16
    for it in range(2):
        dev, n = pb.synth_generate(1920, 1080, 4, iteration=it)
        pb.profile_enable(True)
        pb.profile_collect()
        pb.vertex_pass(g[0], g[1], g[2], None, dev, n, mode=pb.MODE_ATOMIC)
        pb.end_frame_all(g)
        assert gu.launched("k_vertex_pass_tiled")
        pb.profile_enable(False)
        host = dev.cpu().numpy()
        del dev
        po.vertex_pass_ref(r[0], r[1], r[2], None, host, n, deterministic=True, threads=threads)
        for s in r:
            s.end_frame()
        for a, b in zip(g, r):
            gu.assert_slots_close(a.slots(), b.slots(), rtol=1e-9, atol=1e-300)
            _ref_stats_equal(a, b.stats())
