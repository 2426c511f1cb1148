"""Pins the C restatement (oracle/pstf_oracle.c) against the UNMODIFIED reference field engine
compiled from /root/reference into oracle/_ref (CPU only).  Everything is compared bitwise:
keys, levels, slot arrays (occupancy, probe placement, values, counters, ages), query results,
stats and snapshots.  Skipped when oracle/_ref was not built (e.g. on a GPU box)."""
import numpy as np
import pytest

import inputs
import pyoracle as po
import restore_cases as rc

pytestmark = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")


def _cfgs():
    return [po.Config.make(capacity_log2=12, base_cell_size=0.5, max_level=4),
            po.Config.make(capacity_log2=18, base_cell_size=inputs.BASE_CORNELL, max_level=4),
            po.Config.make(capacity_log2=10, base_cell_size=0.01, max_level=6, level_select_k=3.0)]


def _key_arrays_equal(a, b):
    for f in ("level", "cell", "dir", "checksum"):
        np.testing.assert_array_equal(a[f], b[f], err_msg=f)


@pytest.mark.parametrize("ci", range(3))
def test_keys_bitwise(ci):
    cfg = _cfgs()[ci]
    o, r = po.OracleStore(cfg), po.RefStore(cfg)
    rng = np.random.default_rng(1234 + ci)
    n = 60000
    pos = np.concatenate([inputs.random_positions(rng, n), inputs.special_positions()])
    d_struct = inputs.structured_dirs()
    d_spec = inputs.special_dirs()
    d = np.concatenate([inputs.random_dirs(rng, n), d_struct, d_spec])
    pos = np.concatenate([pos, rng.uniform(-3, 3, size=(len(d) - len(pos), 3))])
    for level in range(0, cfg.max_level + 1):
        lv = np.full(len(d), level, np.int32)
        _key_arrays_equal(o.keys_for(pos, d, lv), r.keys_for(pos, d, lv))


@pytest.mark.parametrize("ci", range(3))
def test_select_level_bitwise(ci):
    cfg = _cfgs()[ci]
    o, r = po.OracleStore(cfg), po.RefStore(cfg)
    rng = np.random.default_rng(99 + ci)
    fp = np.concatenate([inputs.level_footprints(cfg.base_cell_size, cfg.level_select_k),
                         inputs.random_footprints(rng, 50000, cfg.base_cell_size)])
    np.testing.assert_array_equal(o.select_levels(fp), r.select_levels(fp))


def _random_session(stores, rng, frames, n_keys, ops_per_frame, levels=(0, 1, 2)):
    """Drive identical scalar call sequences into every store; yield after each endFrame."""
    s0 = stores[0]
    pos = rng.uniform(-4, 4, size=(n_keys, 3))
    dirs = inputs.random_dirs(rng, n_keys)
    lv = rng.choice(levels, size=n_keys).astype(np.int32)
    keys = [s0.key_for(pos[i], dirs[i], lv[i]) for i in range(n_keys)]
    for f in range(frames):
        hot = rng.choice(n_keys, size=max(1, n_keys // 2), replace=False)
        for _ in range(ops_per_frame):
            i = int(rng.choice(hot))
            op = rng.random()
            if op < 0.45:
                w = float(rng.choice([1.0, 0.5, 2.0, 0.0, -1.0, np.nan, np.inf]))
                for s in stores:
                    s.increment_counter(keys[i], w)
            elif op < 0.9:
                v = rng.uniform(0, 3, size=3)
                if rng.random() < 0.05:
                    v[rng.integers(3)] = np.nan
                w = float(rng.choice([1.0, 1.0, 0.25, 0.0, -0.5]))
                for s in stores:
                    s.accumulate(keys[i], v, w)
            else:
                j = int(rng.integers(n_keys))
                res = [s.query_from_level(pos[j], dirs[j], int(lv[j])) for s in stores]
                assert all(x == res[0] for x in res[1:])
        if rng.random() < 0.1:
            for s in stores:
                s.invalidate()
        elif rng.random() < 0.1:
            lo, hi = rng.uniform(-4, 0, 3), rng.uniform(0, 4, 3)
            for s in stores:
                s.invalidate(lo, hi)
        for s in stores:
            s.end_frame()
        yield f


def _slots_equal(a, b):
    for f in po.SLOT_DTYPE.names:
        np.testing.assert_array_equal(np.ascontiguousarray(a[f]).view(np.uint8),
                                      np.ascontiguousarray(b[f]).view(np.uint8), err_msg=f)


@pytest.mark.parametrize("cap,window,evict", [(4, 16, 2), (6, 4, 2), (8, 32, 3), (10, 8, 64)])
def test_scalar_sessions_bitwise(cap, window, evict):
    cfg = po.Config.make(capacity_log2=cap, base_cell_size=0.5, probe_window=window,
                         evict_age_frames=evict, t_max=8.0)
    o, r = po.OracleStore(cfg), po.RefStore(cfg)
    rng = np.random.default_rng(cap * 100 + window)
    n_keys = int((1 << cap) * 1.3)
    for _ in _random_session([o, r], rng, frames=8, n_keys=n_keys, ops_per_frame=6 * n_keys):
        _slots_equal(o.slots(), r.slots())
        assert o.stats() == r.stats()
        np.testing.assert_array_equal(o.weighted_mean(), r.weighted_mean())


def _random_updates(store, rng, n, n_keys):
    pos = rng.uniform(-4, 4, size=(n_keys, 3))
    dirs = inputs.random_dirs(rng, n_keys)
    lv = rng.integers(0, 3, size=n_keys).astype(np.int32)
    keys = store.keys_for(pos, dirs, lv)
    u = np.zeros(n, po.UPDATE_DTYPE)
    idx = rng.integers(0, n_keys, size=n)
    u["key"] = keys[idx]
    u["is_counter"] = rng.random(n) < 0.4
    u["value"] = rng.uniform(0, 2, size=(n, 3))
    u["w"] = rng.choice([1.0, 0.5, 2.0, 0.0], size=n)
    bad = rng.random(n) < 0.01
    u["w"][bad] = np.nan
    return u


@pytest.mark.parametrize("cap,window", [(5, 8), (8, 32), (12, 32)])
def test_queue_apply_bitwise(cap, window):
    cfg = po.Config.make(capacity_log2=cap, base_cell_size=0.5, probe_window=window,
                         evict_age_frames=2)
    o, r = po.OracleStore(cfg), po.RefStore(cfg)
    rng = np.random.default_rng(7 + cap)
    n_keys = int((1 << cap) * 1.2)
    for f in range(5):
        u = _random_updates(o, rng, 4 * n_keys, n_keys)
        perm = rng.permutation(len(u))
        o.queue_apply(u)
        r.queue_apply(u[perm])
        for s in (o, r):
            s.end_frame()
        _slots_equal(o.slots(), r.slots())
        assert o.stats() == r.stats()


@pytest.mark.parametrize("deterministic", [True, False])
@pytest.mark.parametrize("cap,mult", [(10, 8.0), (11, 30.0), (17, 1.0)])
def test_vertex_pass_bitwise(deterministic, cap, mult):
    """Restated onVertex (oracle) == reference FieldStore driven by the public-API replay.
    Small tables force drops and eviction; base multipliers spread the levels 0..4."""
    base = inputs.BASE_CORNELL * mult
    mk = lambda kind: po.Config.make(kind=kind, capacity_log2=cap, base_cell_size=base,
                                     evict_age_frames=2)
    o = [po.OracleStore(mk(k)) for k in (0, 1, 3, 2)]
    r = [po.RefStore(mk(k)) for k in (0, 1, 3, 2)]
    for it in range(4):
        buf, n = po.synth_generate(48, 27, 4, seed=0x5EED, iteration=it)
        po.vertex_pass_oracle(*o, buf, n, deterministic=deterministic)
        po.vertex_pass_ref(*r, buf, n, deterministic=deterministic, threads=1)
        for a, b in zip(o, r):
            a.end_frame()
            b.end_frame()
            _slots_equal(a.slots(), b.slots())
            assert a.stats() == b.stats()


def test_deterministic_ref_threads_equal():
    """Deterministic mode of the reference is worker-count independent (acceptance crit. 10);
    our oracle matches it at any worker count."""
    base = inputs.BASE_CORNELL
    mk = lambda kind: po.Config.make(kind=kind, capacity_log2=14, base_cell_size=base)
    o = [po.OracleStore(mk(k)) for k in (0, 1, 3)] + [None]
    r = [po.RefStore(mk(k)) for k in (0, 1, 3)] + [None]
    for it in range(2):
        buf, n = po.synth_generate(40, 30, 4, iteration=it)
        po.vertex_pass_oracle(*o, buf, n, deterministic=True)
        po.vertex_pass_ref(*r, buf, n, deterministic=True, threads=4, chunk=37)
        for a, b in zip(o[:3], r[:3]):
            a.end_frame()
            b.end_frame()
            _slots_equal(a.slots(), b.slots())


def test_snapshot_records_match_reference_file(tmp_path):
    cfg = po.Config.make(capacity_log2=10, base_cell_size=0.5)
    o, r = po.OracleStore(cfg), po.RefStore(cfg)
    rng = np.random.default_rng(5)
    u = _random_updates(o, rng, 3000, 500)
    o.queue_apply(u)
    r.queue_apply(u)
    o.end_frame()
    r.end_frame()
    r.dump_snapshot(str(tmp_path / "a.snap"))
    kind, recs = po.read_snapshot(str(tmp_path / "a.snap"))
    mine = o.snapshot()
    assert kind == 0 and len(recs) == len(mine)
    for f in po.SNAP_DTYPE.names:
        np.testing.assert_array_equal(recs[f], mine[f])


@pytest.mark.parametrize("cap,window,prefill", [(13, 32, False), (10, 8, False), (11, 32, True),
                                                (8, 4, True)])
def test_restore_matches_reference_insert(cap, window, prefill):
    """po_restore (the oracle's snapshot restore) == restore through the reference's own
    findOrInsertSlot (oracle/ref_shim.cpp pr_restore): slots and counters bitwise, including
    drops (small tables), duplicate keys (the last in key order wins) and restores into a
    store that already holds cells."""
    rng = np.random.default_rng(cap * 7 + window)
    recs = rc.restore_records(rng)
    cfg = po.Config.make(capacity_log2=cap, base_cell_size=0.5, probe_window=window)
    o, r = po.OracleStore(cfg), po.RefStore(cfg)
    if prefill:
        u = rc.random_updates(o, rng, 2000, 700)
        for s in (o, r):
            s.queue_apply(u)
            s.end_frame()
    o.restore(recs)
    r.restore(recs)
    _slots_equal(o.slots(), r.slots())
    assert o.stats() == r.stats()
    if cap == 13 and not prefill:  # no drops: the snapshot is the input, last duplicate wins
        assert o.stats()["dropped"] == 0
        snap, want = o.snapshot(), rc.expected_restore(recs)
        for f in po.SNAP_DTYPE.names:  # per field: the records' padding bytes are unspecified
            np.testing.assert_array_equal(np.ascontiguousarray(snap[f]).view(np.uint8),
                                          np.ascontiguousarray(want[f]).view(np.uint8), err_msg=f)


# ---------------------------------------------------------------- ModelStore<DirGrid> (§8f row 2)
def _model_equal(a, b):
    ea, wa, aa = a.dump()
    eb, wb, ab = b.dump()
    assert len(ea) == len(eb)
    for f in po.MODEL_ENTRY_DTYPE.names:
        np.testing.assert_array_equal(np.ascontiguousarray(ea[f]).view(np.uint8),
                                      np.ascontiguousarray(eb[f]).view(np.uint8), err_msg=f)
    np.testing.assert_array_equal(wa.view(np.uint64), wb.view(np.uint64))
    np.testing.assert_array_equal(aa.view(np.uint64), ab.view(np.uint64))


@pytest.mark.skipif(not po.model_ref_available(), reason="oracle/_ref model store not built")
@pytest.mark.parametrize("res,t_max,min_samples", [(16, 64.0, 32), (5, 2.0, 1), (1, np.inf, 4)])
def test_model_store_matches_reference(res, t_max, min_samples):
    """po_model_* (C restatement) == the reference's ModelStore/DirGrid compiled in place: every
    entry (cOld, cNew, records, recordCount, warm, total), weights and accumulators bitwise over
    apply/endFrame frames, then pdf and sample of warm models bitwise."""
    import model_cases as mc
    rng = np.random.default_rng(res * 31 + min_samples)
    o = po.OracleModelStore(res, t_max, min_samples)
    r = po.RefModelStore(res, t_max, min_samples)
    for frame in range(4):
        k, u, v, c, keys = mc.model_records(rng, 6000, 400)
        o.apply(k, u, v, c)
        r.apply(k, u, v, c)
        _model_equal(o, r)  # accumulators before the blend
        o.end_frame()
        r.end_frame()
        _model_equal(o, r)
    q, u, v = mc.probe_points(rng, keys, 3000)
    po_, fo = o.pdf(q, u, v)
    pr_, fr = r.pdf(q, u, v)
    np.testing.assert_array_equal(fo, fr)
    np.testing.assert_array_equal(po_.view(np.uint64), pr_.view(np.uint64))
    so = o.sample(q, u, v)
    sr = r.sample(q, u, v)
    for a, b in zip(so, sr):
        np.testing.assert_array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
    assert fo.sum() > 100


@pytest.mark.skipif(not po.model_ref_available(), reason="oracle/_ref model store not built")
@pytest.mark.parametrize("leaves,tsplit,t_max", [(64, 4.0, 64.0), (8, 1.5, 3.0), (2, 1.01, np.inf)])
def test_kdtree_model_store_matches_reference(leaves, tsplit, t_max):
    """SphericalKdTree kind (models.cpp:96-298): node probabilities, accumulators, masses and the
    split-collapse topology bitwise against the reference over frames with a hot corner, then
    pdf and sample."""
    import model_cases as mc
    rng = np.random.default_rng(leaves * 7)
    o = po.OracleModelStore(16, t_max, 4, kind=1, leaves=leaves, tsplit=tsplit)
    r = po.RefModelStore(16, t_max, 4, kind=1, leaves=leaves, tsplit=tsplit)
    for frame in range(6):
        k, u, v, c, keys = mc.model_records(rng, 5000, 150, skew=3.0)
        o.apply(k, u, v, c)
        r.apply(k, u, v, c)
        _model_equal(o, r)
        o.end_frame()
        r.end_frame()
        _model_equal(o, r)
        (ti, tf), (ri, rf) = o.dump_tree(), r.dump_tree()
        np.testing.assert_array_equal(ti, ri)
        np.testing.assert_array_equal(tf.view(np.uint64), rf.view(np.uint64))
    moved = (ti[:, :, 4] != po.OracleModelStore(16, t_max, 4, kind=1, leaves=leaves,
                                                tsplit=tsplit)._initial_parents(leaves)).any(1)
    q, u, v = mc.probe_points(rng, keys, 3000)
    po_, fo = o.pdf(q, u, v)
    pr_, fr = r.pdf(q, u, v)
    np.testing.assert_array_equal(fo, fr)
    np.testing.assert_array_equal(po_.view(np.uint64), pr_.view(np.uint64))
    for a, b in zip(o.sample(q, u, v), r.sample(q, u, v)):
        np.testing.assert_array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
    assert fo.sum() > 50 and (moved.sum() > 0 or leaves == 2)  # warm; split-collapse happened


@pytest.mark.skipif(not po.model_ref_available(), reason="oracle/_ref model store not built")
@pytest.mark.parametrize("comps,alpha,skew", [(4, 0.7, 2.0), (3, 0.95, 1.0), (1, 0.6, 3.0)])
def test_gmm_model_store_matches_reference(comps, alpha, skew):
    """Gmm kind (models.cpp:427-702: batch E-step by prefix sums, M-step with eigenvalue clamps
    and reseeding): the C restatement uses the same libm as the reference, so the whole state
    (weights, means, covariances, statistics, cache, step index, underflows, reseeds), pdf and
    sample agree bitwise."""
    import model_cases as mc
    rng = np.random.default_rng(comps * 13 + int(alpha * 100))
    o = po.OracleModelStore(16, 64.0, 4, kind=2, comps=comps, alpha_em=alpha)
    r = po.RefModelStore(16, 64.0, 4, kind=2, comps=comps, alpha_em=alpha)
    for frame in range(5):
        k, u, v, c, keys = mc.model_records(rng, 4000, 120, skew=skew)
        o.apply(k, u, v, c)
        r.apply(k, u, v, c)
        o.end_frame()
        r.end_frame()
        _model_equal(o, r)
    q, u, v = mc.probe_points(rng, keys, 2000)
    us = rng.random(len(q))
    po_, fo = o.pdf(q, u, v)
    pr_, fr = r.pdf(q, u, v)
    np.testing.assert_array_equal(fo, fr)
    np.testing.assert_array_equal(po_.view(np.uint64), pr_.view(np.uint64))
    for a, b in zip(o.sample(q, u, v, us), r.sample(q, u, v, us)):
        np.testing.assert_array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
    assert fo.sum() > 50



@pytest.mark.parametrize("extreme", [False, True])
def test_crafted_stream_oracle_vs_reference(extreme):
    """the adversarial streams of tests/crafted.py (escapes, NaN/inf values, ratio <= 0,
    boundary-hugging keys) replayed through the C restatement and the reference: bitwise"""
    import crafted
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    base = (12.0 ** 0.5) / 256.0
    kinds = (po.KIND_LO, po.KIND_LOE, po.KIND_FLI, po.KIND_LI)
    ref = [po.RefStore(po.Config.make(kind=k, capacity_log2=13, base_cell_size=base)) for k in kinds]
    orc = [po.OracleStore(po.Config.make(kind=k, capacity_log2=13, base_cell_size=base)) for k in kinds]
    for f in range(4):
        buf, n = po.synth_generate(40, 30, 4, iteration=f)
        crafted.mutate(buf, n, seed=77 + f, base=base, extreme=extreme)
        masks = (1 + f % 7, 1 + (2 * f + 3) % 7)
        po.vertex_pass_ref(ref[0], ref[1], ref[2], ref[3], buf, n, masks[0], masks[1],
                           deterministic=True)
        po.vertex_pass_oracle(orc[0], orc[1], orc[2], orc[3], buf, n, masks[0], masks[1],
                              deterministic=True)
        for s in ref + orc:
            s.end_frame()
        for a, b in zip(ref, orc):
            assert a.slots().tobytes() == b.slots().tobytes(), f
            assert a.stats() == b.stats()
    assert sum(s.stats()["rejected"] for s in ref) > 0
