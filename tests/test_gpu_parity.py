"""GPU parity: the B200 field cache (through the C ABI) against the CPU oracle and, when built,
the reference itself (oracle/_ref).  Keys, levels, slot occupancy, probe placement, counters,
ages and query results are compared bitwise; ORDERED/SEQUENTIAL modes are bitwise in values
too; ATOMIC-mode values must agree within rtol 1e-9 (north star: 1e-5)."""
import os

import numpy as np
import pytest

import gpu_util as gu
import inputs
import pyoracle as po
import restore_cases as rc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2005_07547_b200 as pb  # noqa: E402


def _checker(cfg):
    return po.RefStore(cfg) if po.ref_available() else po.OracleStore(cfg)


def _pcfg(cfg: po.Config) -> pb.FieldStoreConfig:
    return pb.FieldStoreConfig(kind=cfg.kind, capacity_log2=cfg.capacity_log2,
                               max_level=cfg.max_level, base_cell_size=cfg.base_cell_size,
                               level_select_k=cfg.level_select_k, t_max=cfg.t_max,
                               blend=cfg.blend, technique_mask=cfg.technique_mask,
                               probe_window=cfg.probe_window,
                               evict_age_frames=cfg.evict_age_frames)


# ------------------------------------------------------------------ K1 keygen / select_level
@pytest.mark.parametrize("base", [0.5, inputs.BASE_CORNELL])
def test_keys_device_bitwise(base):
    cfg = po.Config.make(capacity_log2=10, base_cell_size=base)
    ref = _checker(cfg)
    g = pb.FieldStore(_pcfg(cfg))
    rng = np.random.default_rng(11)
    d = np.concatenate([inputs.random_dirs(rng, 300000), inputs.boundary_dirs(rng, 200000),
                        inputs.structured_dirs(), inputs.special_dirs(),
                        inputs.special_dirs_extra()])
    n = len(d)
    pos = np.concatenate([inputs.random_positions(rng, n - 8), inputs.special_positions()])
    for level in range(cfg.max_level + 1):
        lv = np.full(n, level, np.int32)
        got = g.key_for_batch(torch.from_numpy(pos), torch.from_numpy(d), torch.from_numpy(lv))
        got = got.cpu().numpy().view(po.KEY_DTYPE).reshape(n)
        want = ref.keys_for(pos, d, lv)
        for f in ("level", "cell", "dir", "checksum"):
            bad = (got[f] != want[f]).reshape(n, -1).any(1)
            assert not bad.any(), (level, f, np.nonzero(bad)[0][:10])


def test_select_level_device_bitwise():
    cfg = po.Config.make(capacity_log2=10, base_cell_size=inputs.BASE_CORNELL)
    ref = _checker(cfg)
    g = pb.FieldStore(_pcfg(cfg))
    rng = np.random.default_rng(12)
    fp = np.concatenate([inputs.level_footprints(cfg.base_cell_size),
                         inputs.random_footprints(rng, 500000, cfg.base_cell_size)])
    got = g.select_level_batch(torch.from_numpy(fp)).cpu().numpy()
    np.testing.assert_array_equal(got, ref.select_levels(fp))


# ------------------------------------------------------------------ scalar call sequences
def _session(stores, rng, frames, n_keys, ops, levels=(0, 1, 2), check=None):
    pos = rng.uniform(-4, 4, size=(n_keys, 3))
    dirs = inputs.random_dirs(rng, n_keys)
    lv = rng.choice(levels, size=n_keys).astype(np.int32)
    o = stores[0]
    keys = [o.key_for(pos[i], dirs[i], lv[i]) for i in range(n_keys)]
    gkeys = [pb.SpatioDirectionalKey(k.level, tuple(k.cell), tuple(k.dir), k.checksum)
             for k in keys]
    g = stores[1]
    for f in range(frames):
        hot = rng.choice(n_keys, size=max(1, n_keys // 2), replace=False)
        for _ in range(ops):
            i = int(rng.choice(hot))
            if rng.random() < 0.45:
                w = float(rng.choice([1.0, 0.5, 2.0, 0.0, -1.0, np.nan]))
                o.increment_counter(keys[i], w)
                g.incrementCounter(gkeys[i], w)
            else:
                v = rng.uniform(0, 3, size=3)
                if rng.random() < 0.05:
                    v[0] = np.nan
                w = float(rng.choice([1.0, 0.25, 0.0]))
                o.accumulate(keys[i], v, w)
                g.accumulate(gkeys[i], v, w)
        if rng.random() < 0.15:
            lo, hi = rng.uniform(-4, 0, 3), rng.uniform(0, 4, 3)
            o.invalidate(lo, hi)
            g.invalidate((lo, hi))
        o.end_frame()
        g.end_frame()
        if check:
            check(f, pos, dirs, lv)


@pytest.mark.parametrize("cap,window,evict", [(4, 16, 2), (6, 4, 2), (9, 32, 3)])
def test_scalar_sequence_bitwise(cap, window, evict):
    """SEQUENTIAL mode == the reference's scalar incrementCounter/accumulate sequence."""
    cfg = po.Config.make(capacity_log2=cap, base_cell_size=0.5, probe_window=window,
                         evict_age_frames=evict, t_max=8.0)
    o = po.OracleStore(cfg)
    g = pb.FieldStore(_pcfg(cfg))
    rng = np.random.default_rng(cap * 7 + window)
    n_keys = int((1 << cap) * 1.3)

    def check(f, pos, dirs, lv):
        gu.assert_slots_bitwise(g.slots(), o.slots())
        st, so = g.stats(), o.stats()
        for k in ("frame", "rejected", "dropped", "internal_errors", "live"):
            assert st[k] == so[k], (f, k, st[k], so[k])
        v, ok, fb, ol = g.query_batch(torch.from_numpy(pos), torch.from_numpy(dirs),
                                      level=torch.from_numpy(lv))
        rv, rok, rfb, rol = o.query_batch(pos, dirs, level=lv)
        np.testing.assert_array_equal(ok.cpu().numpy(), rok)
        np.testing.assert_array_equal(fb.cpu().numpy(), rfb)
        np.testing.assert_array_equal(ol.cpu().numpy(), rol)
        np.testing.assert_array_equal(gu.bits(v.cpu().numpy().T), gu.bits(rv))

    _session([o, g], rng, frames=6, n_keys=n_keys, ops=5 * n_keys, check=check)


def _random_updates(store, rng, n, n_keys, levels=3):
    pos = rng.uniform(-4, 4, size=(n_keys, 3))
    dirs = inputs.random_dirs(rng, n_keys)
    lv = rng.integers(0, levels, size=n_keys).astype(np.int32)
    keys = store.keys_for(pos, dirs, lv)
    u = np.zeros(n, po.UPDATE_DTYPE)
    idx = rng.integers(0, n_keys, size=n)
    u["key"] = keys[idx]
    u["is_counter"] = rng.random(n) < 0.4
    u["value"] = rng.uniform(0, 2, size=(n, 3))
    u["w"] = rng.choice([1.0, 0.5, 2.0, 0.0], size=n)
    u["w"][rng.random(n) < 0.01] = np.nan
    return u


def _apply_gpu(g, u, mode):
    keys = torch.from_numpy(np.ascontiguousarray(u["key"]).view(np.int32).reshape(-1, 7).copy())
    v = torch.from_numpy(np.ascontiguousarray(u["value"].T))
    w = torch.from_numpy(np.ascontiguousarray(u["w"]))
    isc = torch.from_numpy(u["is_counter"].astype(np.uint8))
    g.apply(keys, v, w, isc, mode)


@pytest.mark.parametrize("mode", ["ordered", "sequential"])
def test_inexact_counter_weights_bitwise(mode):
    """Counter weights that are not whole numbers (uniform in (0, 3)) make the frame's Σc_new
    depend on summation order; with t_max = 2 the c_old cap (T^2 - T) * mean c_new binds on most
    slots, so the committed state is bitwise the reference's only if the mean is summed in
    slot order (field.cpp:201-213)."""
    cfg = po.Config.make(capacity_log2=12 if mode == "ordered" else 9, base_cell_size=0.5,
                         probe_window=32, evict_age_frames=3, t_max=2.0)
    o = po.OracleStore(cfg)
    g = pb.FieldStore(_pcfg(cfg))
    rng = np.random.default_rng(77)
    if mode == "ordered":
        n_keys = 3000
        for f in range(5):
            u = _random_updates(o, rng, 6 * n_keys, n_keys)
            u["w"] = rng.uniform(0.0, 3.0, size=len(u))
            o.queue_apply(u)
            _apply_gpu(g, u[rng.permutation(len(u))], pb.MODE_ORDERED)
            o.end_frame()
            g.end_frame()
            gu.assert_slots_bitwise(g.slots(), o.slots())
        return
    # SEQUENTIAL: the scalar calls (the facade flushes them in submission order)
    n_keys = 400
    pos = rng.uniform(-4, 4, size=(n_keys, 3))
    dirs = inputs.random_dirs(rng, n_keys)
    keys = [o.key_for(pos[i], dirs[i], 0) for i in range(n_keys)]
    gkeys = [pb.SpatioDirectionalKey(k.level, tuple(k.cell), tuple(k.dir), k.checksum)
             for k in keys]
    for f in range(5):
        for _ in range(3 * n_keys):
            i = int(rng.integers(n_keys))
            w = float(rng.uniform(0.0, 3.0))
            if rng.random() < 0.5:
                o.increment_counter(keys[i], w)
                g.incrementCounter(gkeys[i], w)
            else:
                v = rng.uniform(0, 3, size=3)
                o.accumulate(keys[i], v, w)
                g.accumulate(gkeys[i], v, w)
        o.end_frame()
        g.end_frame()
        gu.assert_slots_bitwise(g.slots(), o.slots())


@pytest.mark.parametrize("cap,window", [(5, 8), (8, 32), (14, 32)])
def test_queue_apply_ordered_bitwise(cap, window):
    """ORDERED mode == FieldUpdateQueue::apply (field.cpp:396-420), values bitwise."""
    cfg = po.Config.make(capacity_log2=cap, base_cell_size=0.5, probe_window=window,
                         evict_age_frames=2)
    o = po.OracleStore(cfg)
    g = pb.FieldStore(_pcfg(cfg))
    rng = np.random.default_rng(100 + cap)
    n_keys = int((1 << cap) * 1.2)
    for f in range(5):
        u = _random_updates(o, rng, 4 * n_keys, n_keys)
        o.queue_apply(u)
        _apply_gpu(g, u[rng.permutation(len(u))], pb.MODE_ORDERED)
        gu.assert_slots_bitwise(g.slots(), o.slots(), ("checksum", "level", "cell", "dir",
                                                       "accum", "c_new", "last_touched"))
        o.end_frame()
        g.end_frame()
        gu.assert_slots_bitwise(g.slots(), o.slots())
        st, so = g.stats(), o.stats()
        for k in ("frame", "rejected", "dropped", "internal_errors", "live"):
            assert st[k] == so[k], (f, k)


@pytest.mark.parametrize("cap,window", [(5, 8), (14, 32)])
def test_apply_atomic_occupancy_bitwise(cap, window):
    """ATOMIC mode: placement/occupancy/ages/counters bitwise, values to 1e-12 relative."""
    cfg = po.Config.make(capacity_log2=cap, base_cell_size=0.5, probe_window=window,
                         evict_age_frames=2)
    o = po.OracleStore(cfg)
    g = pb.FieldStore(_pcfg(cfg))
    rng = np.random.default_rng(200 + cap)
    n_keys = int((1 << cap) * 1.2)
    for f in range(5):
        u = _random_updates(o, rng, 4 * n_keys, n_keys)
        o.queue_apply(u)
        _apply_gpu(g, u, pb.MODE_ATOMIC)
        o.end_frame()
        g.end_frame()
        gu.assert_slots_close(g.slots(), o.slots(), rtol=1e-12)
        st, so = g.stats(), o.stats()
        for k in ("frame", "rejected", "dropped", "internal_errors", "live"):
            assert st[k] == so[k], (f, k)


# ------------------------------------------------------------------ fused vertex pass (K5)
def _vertex_stores(cap, base, mk_gpu=True, li=False, evict=64):
    kinds = (po.KIND_LO, po.KIND_LOE, po.KIND_FLI) + ((po.KIND_LI,) if li else ())
    cfgs = [po.Config.make(kind=k, capacity_log2=cap, base_cell_size=base, evict_age_frames=evict)
            for k in kinds]
    o = [po.OracleStore(c) for c in cfgs]
    g = [pb.FieldStore(_pcfg(c)) for c in cfgs]
    if not li:
        o.append(None)
        g.append(None)
    return o, g


@pytest.mark.parametrize("mode", ["atomic", "ordered"])
@pytest.mark.parametrize("cap,mult,li,evict", [(10, 8.0, False, 2), (12, 30.0, True, 64),
                                               (16, 1.0, False, 64), (18, 2.0, True, 3)])
def test_vertex_pass_vs_oracle(mode, cap, mult, li, evict):
    o, g = _vertex_stores(cap, inputs.BASE_CORNELL * mult, li=li, evict=evict)
    gm = pb.MODE_ATOMIC if mode == "atomic" else pb.MODE_ORDERED
    for it in range(5):
        buf, n = pb.synth_generate(96, 54, 4, iteration=it)
        pb.vertex_pass(*g, buf, n, mode=gm)
        po.vertex_pass_oracle(*o, buf.cpu().numpy(), n, deterministic=True)
        for a, b in zip(g, o):
            if a is None:
                continue
            a.end_frame()
            b.end_frame()
            if mode == "ordered":
                gu.assert_slots_bitwise(a.slots(), b.slots())
            else:
                gu.assert_slots_close(a.slots(), b.slots(), rtol=1e-9)
            st, so = a.stats(), b.stats()
            for k in ("frame", "rejected", "dropped", "internal_errors", "live"):
                assert st[k] == so[k], (it, k, st[k], so[k])


@pytest.mark.parametrize("w,h,b", [(97, 53, 4), (33, 21, 3), (128, 1, 4), (5, 3, 2)])
def test_vertex_pass_shapes(w, h, b):
    """Tail tiles (n % 128 != 0), unaligned SoA segments (odd n -> non-TMA kernel) and tiny
    streams all give the oracle's occupancy/counters and values (ATOMIC)."""
    o, g = _vertex_stores(14, inputs.BASE_CORNELL * 6.0, li=True, evict=2)
    for it in range(3):
        buf, n = pb.synth_generate(w, h, b, iteration=it)
        pb.vertex_pass(*g, buf, n, mode=pb.MODE_ATOMIC)
        po.vertex_pass_oracle(*o, buf.cpu().numpy(), n, deterministic=True)
        for a, c in zip(g, o):
            a.end_frame()
            c.end_frame()
            gu.assert_slots_close(a.slots(), c.slots(), rtol=1e-9)
            st, so = a.stats(), c.stats()
            for k in ("frame", "rejected", "dropped", "internal_errors", "live"):
                assert st[k] == so[k], (it, k, st[k], so[k])


def test_vertex_pass_field_layouts():
    """The uniformly strided buffer (one 2-D tensor-map copy per tile) and the same fields
    scattered at irregular offsets (35 per-field bulk copies) give the same occupancy,
    counters and values (ATOMIC), and both match the oracle."""
    import torch
    o, g1 = _vertex_stores(14, inputs.BASE_CORNELL * 6.0, li=True, evict=2)
    _, g2 = _vertex_stores(14, inputs.BASE_CORNELL * 6.0, li=True, evict=2)
    for it in range(3):
        buf, n = pb.synth_generate(128, 72, 4, iteration=it)
        f = buf[:34 * n].view(34, n)
        stride = n + 48  # fields in reverse order with an irregular gap
        scat = torch.zeros(34 * stride + 64, dtype=torch.float64, device="cuda")
        fields = []
        for k in range(34):
            off = (33 - k) * stride + (16 if k % 3 == 0 else 0)
            scat[off:off + n] = f[k]
            fields.append(scat[off:off + n])
        flags = buf[34 * n:].view(torch.int32)[:n].clone()
        pb.vertex_pass(*g1, buf, n, mode=pb.MODE_ATOMIC)
        pb.vertex_pass(*g2, None, n, mode=pb.MODE_ATOMIC,
                       soa=pb.vertex_soa_from_fields(fields, flags))
        po.vertex_pass_oracle(*o, buf.cpu().numpy(), n, deterministic=True)
        for a, b, c in zip(g1, g2, o):
            a.end_frame()
            b.end_frame()
            c.end_frame()
            gu.assert_slots_close(a.slots(), c.slots(), rtol=1e-9)
            gu.assert_slots_close(b.slots(), c.slots(), rtol=1e-9)
            for k in ("rejected", "dropped", "live"):
                assert a.stats()[k] == b.stats()[k] == c.stats()[k]


@pytest.mark.parametrize("mode", ["atomic", "ordered"])
def test_vertex_pass_cv_fused(mode):
    """pstf_vertex_pass_cv == pstf_cv_lookup on the frame-start table (bitwise) followed by
    pstf_vertex_pass (same stores afterwards), on both the fused tiled kernel (ATOMIC) and the
    separate-kernel path (ORDERED)."""
    gm = pb.MODE_ATOMIC if mode == "atomic" else pb.MODE_ORDERED
    _, g1 = _vertex_stores(14, inputs.BASE_CORNELL * 6.0, li=True, evict=2)
    _, g2 = _vertex_stores(14, inputs.BASE_CORNELL * 6.0, li=True, evict=2)
    for it in range(4):
        buf, n = pb.synth_generate(128, 72, 4, iteration=it % 2)
        ref_val, ref_ok = pb.cv_lookup(g2[1], buf, n)  # read-only: the frame-start table
        pb.vertex_pass(*g1, buf, n, mode=gm)
        val, ok = pb.vertex_pass_cv(*g2, buf, n, mode=gm)
        np.testing.assert_array_equal(ok.cpu().numpy().astype(bool), ref_ok.cpu().numpy())
        np.testing.assert_array_equal(gu.bits(val.cpu().numpy()), gu.bits(ref_val.cpu().numpy()))
        if it:
            assert ok.cpu().numpy().mean() > 0.3
        for a, b in zip(g1, g2):
            a.end_frame()
            b.end_frame()
            if mode == "ordered":
                gu.assert_slots_bitwise(a.slots(), b.slots())
            else:
                gu.assert_slots_close(a.slots(), b.slots(), rtol=1e-9)


def test_probe_histogram_vs_oracle_slots():
    """pstf_field_probe_histogram == the distances of the oracle's live slots from their homes
    (home = packKeyFields(key) & mask, field.cpp:104), on a crowded table with drops."""
    from shard_cpu_backend import pack
    o, g = _vertex_stores(12, inputs.BASE_CORNELL * 2.0, li=False, evict=64)
    for it in range(3):
        buf, n = pb.synth_generate(96, 54, 4, iteration=it)
        pb.vertex_pass(*g, buf, n, mode=pb.MODE_ATOMIC)
        po.vertex_pass_oracle(*o, buf.cpu().numpy(), n, deterministic=True)
        for a, b in zip(g[:3], o[:3]):
            a.end_frame()
            b.end_frame()
    for a, b in zip(g[:3], o[:3]):
        sl = b.slots()
        mask = len(sl) - 1
        want = np.zeros(33, np.uint64)
        for i in np.nonzero(sl["checksum"])[0]:
            k = (int(sl["level"][i]), *[int(c) for c in sl["cell"][i]], *[int(d) for d in sl["dir"][i]])
            d = (int(i) - (pack(k) & mask)) & mask
            want[min(d, 32)] += 1
        got = a.probe_histogram()
        np.testing.assert_array_equal(got, want)
        assert got.sum() == a.stats()["live"]
    assert any(a.probe_histogram()[1:].sum() > 0 for a in g[:3])  # collisions exercised


def test_red_counter_and_peak():
    """The fused kernel's RED accounting is positive and below the unaggregated bound, and the
    RED peak diagnostic returns a plausible rate."""
    _, g = _vertex_stores(16, inputs.BASE_CORNELL, li=False)
    buf, n = pb.synth_generate(128, 72, 4, iteration=0)
    pb.vertex_pass(*g, buf, n, mode=pb.MODE_ATOMIC)
    pb.vertex_pass(*g, buf, n, mode=pb.MODE_ATOMIC)
    reds = g[0].stats()["reds_total"]
    assert 0 < reds <= 2 * n * 4 * 4
    peak = pb.red_peak(0)
    assert 1e9 < peak < 1e13


def test_deferred_phase2_identical(tmp_path):
    """The deferred phase 2 (pstf_vertex_pass returns after phase 1; endFrame guarded by the
    device-side pending count; other entry points settle first) gives the same stores, stats and
    slot arrays as placing the new keys before returning (PSTF_NO_DEFER=1)."""
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    outs = []
    for env_extra in ({}, {"PSTF_NO_DEFER": "1"}):
        out = str(tmp_path / f"d{len(outs)}.npz")
        env = dict(os.environ, **env_extra)
        r = subprocess.run([sys.executable, os.path.join(here, "defer_probe.py"), out], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        outs.append(np.load(out))
    a, b = outs
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        if k.startswith("slots"):
            sa = a[k].view(pb.SLOT_DTYPE)
            sb = b[k].view(pb.SLOT_DTYPE)
            gu.assert_slots_close(sa, sb, rtol=1e-9)
        else:
            np.testing.assert_array_equal(a[k], b[k])


def test_vertex_pass_matches_reference_replay():
    """Against the reference FieldStore itself (EstimatorRun deterministic-mode replay)."""
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    base = inputs.BASE_CORNELL * 4.0
    cfgs = [po.Config.make(kind=k, capacity_log2=13, base_cell_size=base, evict_age_frames=2)
            for k in (0, 1, 3)]
    r = [po.RefStore(c) for c in cfgs] + [None]
    g = [pb.FieldStore(_pcfg(c)) for c in cfgs] + [None]
    for it in range(4):
        buf, n = pb.synth_generate(80, 45, 4, iteration=it)
        pb.vertex_pass(*g, buf, n, mode=pb.MODE_ORDERED)
        po.vertex_pass_ref(*r, buf.cpu().numpy(), n, deterministic=True, threads=4)
        for a, b in zip(g[:3], r[:3]):
            a.end_frame()
            b.end_frame()
            gu.assert_slots_bitwise(a.slots(), b.slots())


def test_vertex_pass_host_equals_device():
    """pstf_vertex_pass_host (chunked H2D) == pstf_vertex_pass on device data (ORDERED)."""
    base = inputs.BASE_CORNELL * 2
    _, g1 = _vertex_stores(15, base)
    _, g2 = _vertex_stores(15, base)
    for it in range(2):
        buf, n = pb.synth_generate(128, 72, 4, iteration=it)
        host = buf.cpu().pin_memory()
        pb.vertex_pass(*g1, buf, n, mode=pb.MODE_ORDERED)
        pb.vertex_pass_host(*g2, host, n, mode=pb.MODE_ORDERED)
        for a, b in zip(g1[:3], g2[:3]):
            a.end_frame()
            b.end_frame()
            gu.assert_slots_bitwise(a.slots(), b.slots())


@pytest.mark.parametrize("scene", [0, 1])
def test_synth_device_equals_host(scene):
    """the generator is IEEE-exact: device and host streams are bit-identical (scene 1: the
    glossy materials of config 3, Phong lobe sampled as the max of 49 uniforms)"""
    buf, n = pb.synth_generate(64, 36, 4, iteration=3, cam_shift_x=0.1, scene=scene)
    hbuf, hn = po.synth_generate(64, 36, 4, iteration=3, cam_shift_x=0.1, scene=scene)
    assert n == hn
    np.testing.assert_array_equal(gu.bits(buf.cpu().numpy()), gu.bits(hbuf))


# ------------------------------------------------------------------ lookup (K4), CV lookup
def test_query_batch_bitwise_after_frames():
    base = inputs.BASE_CORNELL * 4
    o, g = _vertex_stores(14, base)
    for it in range(3):
        buf, n = pb.synth_generate(64, 36, 4, iteration=it)
        pb.vertex_pass(*g, buf, n, mode=pb.MODE_ORDERED)
        po.vertex_pass_oracle(*o, buf.cpu().numpy(), n, deterministic=True)
        for a, b in zip(g[:3], o[:3]):
            a.end_frame()
            b.end_frame()
    rng = np.random.default_rng(5)
    hb, n = po.synth_generate(64, 36, 4, iteration=9)
    f64, _ = po.soa_views(hb, n)
    pos = f64[0:3].T.copy()
    wo = f64[3:6].T.copy()
    fp = f64[15].copy()
    pos = np.concatenate([pos, rng.uniform(-1, 2, size=(5000, 3))])
    wo = np.concatenate([wo, inputs.random_dirs(rng, 5000)])
    fp = np.concatenate([fp, inputs.random_footprints(rng, 5000, base)])
    for a, b in zip(g[:3], o[:3]):
        v, ok, fb, ol = a.query_batch(torch.from_numpy(pos), torch.from_numpy(wo),
                                      footprint=torch.from_numpy(fp))
        rv, rok, rfb, rol = b.query_batch(pos, wo, fp=fp)
        np.testing.assert_array_equal(ok.cpu().numpy(), rok)
        np.testing.assert_array_equal(fb.cpu().numpy(), rfb)
        np.testing.assert_array_equal(ol.cpu().numpy(), rol)
        np.testing.assert_array_equal(gu.bits(v.cpu().numpy().T), gu.bits(rv))
    # CV lookup at the current vertex == LoE query at (position, wo, footprint)
    dbuf = torch.from_numpy(hb).cuda()
    cv, cok = pb.cv_lookup(g[1], dbuf, n)
    rv, rok, _, _ = o[1].query_batch(f64[0:3].T.copy(), f64[3:6].T.copy(), fp=f64[15].copy())
    np.testing.assert_array_equal(cok.cpu().numpy(), rok)
    np.testing.assert_array_equal(gu.bits(cv.cpu().numpy().T), gu.bits(rv))


# ------------------------------------------------------------------ snapshots / observers
def test_snapshot_file_matches_reference(tmp_path):
    cfg = po.Config.make(capacity_log2=11, base_cell_size=0.5)
    o = _checker(cfg)
    g = pb.FieldStore(_pcfg(cfg))
    rng = np.random.default_rng(9)
    u = _random_updates(po.OracleStore(cfg), rng, 6000, 1500, levels=5)
    o.queue_apply(u)
    _apply_gpu(g, u, pb.MODE_ORDERED)
    o.end_frame()
    g.end_frame()
    gp, rp = str(tmp_path / "g.snap"), str(tmp_path / "r.snap")
    g.dump_snapshot(gp)
    if isinstance(o, po.RefStore):
        o.dump_snapshot(rp)
        assert open(gp, "rb").read() == open(rp, "rb").read()
    kind, recs = pb.read_snapshot(gp)
    mine = g.snapshot()
    ref = o.snapshot()
    assert kind == 0 and len(recs) == len(mine) == len(ref) == g.liveCellCount()
    for f in ("level", "cell", "dir", "checksum", "value", "c_old"):
        np.testing.assert_array_equal(recs[f], ref[f])
        np.testing.assert_array_equal(mine[f], ref[f])
    np.testing.assert_allclose(g.weightedMeanValue(), o.weighted_mean(), rtol=1e-12)
    with pytest.raises(pb.PstfError):
        bad = tmp_path / "bad.snap"
        bad.write_bytes(b"NOTASNAP0000")
        pb.read_snapshot(str(bad))


# ------------------------------------------------------------------ snapshot restore (§8f row 3)
@pytest.mark.parametrize("cap,window,prefill", [(13, 32, False), (10, 8, False), (11, 32, True),
                                                (8, 4, True)])
def test_restore_vs_oracle(cap, window, prefill):
    """pstf_field_restore == the reference's own findOrInsertSlot in ascending key order
    (oracle/ref_shim.cpp pr_restore, pinned in test_oracle_pin): slots, ages, drops bitwise;
    then one more ORDERED frame on top stays bitwise (restored cells blend like native ones)."""
    rng = np.random.default_rng(cap * 7 + window)
    recs = rc.restore_records(rng)
    cfg = po.Config.make(capacity_log2=cap, base_cell_size=0.5, probe_window=window)
    o = _checker(cfg)
    g = pb.FieldStore(_pcfg(cfg))
    if prefill:
        u = rc.random_updates(po.OracleStore(cfg), rng, 2000, 700)
        o.queue_apply(u)
        _apply_gpu(g, u, pb.MODE_ORDERED)
        o.end_frame()
        g.end_frame()
    o.restore(recs)
    g.restore(recs)
    gu.assert_slots_bitwise(g.slots(), o.slots())
    st, so = g.stats(), o.stats()
    for k in ("frame", "rejected", "dropped", "internal_errors", "live"):
        assert st[k] == so[k], k
    u = rc.random_updates(po.OracleStore(cfg), rng, 3000, 1000)
    o.queue_apply(u)
    _apply_gpu(g, u, pb.MODE_ORDERED)
    o.end_frame()
    g.end_frame()
    gu.assert_slots_bitwise(g.slots(), o.slots())
    if cap == 13 and not prefill:
        assert st["dropped"] == 0


def test_snapshot_dump_load_round_trip(tmp_path):
    """dump -> loadSnapshot into a fresh store -> dump: byte-identical files (checkpoint/resume
    of the cache); bad checksums and a wrong field kind are rejected with the store unchanged."""
    cfg = po.Config.make(capacity_log2=14, base_cell_size=0.5)
    g = pb.FieldStore(_pcfg(cfg))
    rng = np.random.default_rng(31)
    for _ in range(3):
        _apply_gpu(g, rc.random_updates(po.OracleStore(cfg), rng, 20000, 6000, levels=5),
                   pb.MODE_ATOMIC)
        g.end_frame()
    a, b = str(tmp_path / "a.snap"), str(tmp_path / "b.snap")
    g.dump_snapshot(a)
    h = pb.FieldStore(_pcfg(cfg))
    h.load_snapshot(a)
    h.dump_snapshot(b)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert h.liveCellCount() == g.liveCellCount() > 5000
    o = _checker(cfg)
    o.restore(pb.read_snapshot(a)[1])
    gu.assert_slots_bitwise(h.slots(), o.slots())
    recs = g.snapshot()
    recs["checksum"][len(recs) // 2] ^= 1
    e = pb.FieldStore(_pcfg(cfg))
    with pytest.raises(pb.PstfError, match="checksum"):
        e.restore(recs)
    assert e.liveCellCount() == 0
    fli = pb.FieldStore(_pcfg(po.Config.make(kind=po.KIND_FLI, capacity_log2=14, base_cell_size=0.5)))
    with pytest.raises(pb.PstfError, match="kind"):
        fli.load_snapshot(a)


# ------------------------------------------------------------------ full-size properties
def test_config2_scale_properties():
    """1920x1080x4 stream at 2^22 slots: ATOMIC and ORDERED give identical occupancy; values
    agree to 1e-9; invariants of a first frame hold exactly (alpha = 1, c_old = c_new)."""
    base = inputs.BASE_CORNELL
    mk = lambda: [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=22,
                                                    base_cell_size=base))
                  for k in (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI)]
    ga, go = mk(), mk()
    for it in range(2):
        buf, n = pb.synth_generate(1920, 1080, 4, iteration=it)
        assert n == 8294400
        pb.vertex_pass(ga[0], ga[1], ga[2], None, buf, n, mode=pb.MODE_ATOMIC)
        pb.vertex_pass(go[0], go[1], go[2], None, buf, n, mode=pb.MODE_ORDERED)
        for a, b in zip(ga, go):
            a.end_frame()
            b.end_frame()
            sa, sb = a.slots(), b.slots()
            gu.assert_slots_close(sa, sb, rtol=1e-9)
            assert a.stats()["live"] == int((sa["checksum"] != 0).sum())
            if it == 0:
                live = sa["checksum"] != 0
                assert (sa["c_old"][live] > 0).all()
                # one Lo counter call per vertex: committed counts add up exactly (no cap hit)
                if a is ga[0] and a.stats()["dropped"] == 0:
                    assert sa["c_old"].sum() == n


def test_repeatability_atomic_occupancy():
    """Two ATOMIC runs of the same frames give bitwise-identical occupancy (deterministic
    placement even though fp64 summation order varies)."""
    base = inputs.BASE_CORNELL
    runs = []
    for _ in range(2):
        gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=18, base_cell_size=base,
                                                evict_age_frames=2))
              for k in (0, 1, 3)]
        for it in range(3):
            buf, n = pb.synth_generate(640, 360, 4, iteration=it)
            pb.vertex_pass(gs[0], gs[1], gs[2], None, buf, n)
            for s in gs:
                s.end_frame()
        runs.append([s.slots() for s in gs])
    for a, b in zip(*runs):
        gu.assert_slots_bitwise(a, b, gu.FIELDS_EXACT)
