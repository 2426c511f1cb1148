"""GPU parity of the model store (ModelStore<DirGrid>, the CV-profile /
guiding store keyed by the field's keys) against the reference's own ModelStore compiled in
place (oracle/_ref/libpstf_model_ref.so) or, without it, the C restatement pinned to it
(tests/test_oracle_pin.py).  Entries, grid weights and accumulators, warm flags, pdf and
sample results are compared bitwise."""
import numpy as np
import pytest

import inputs
import model_cases as mc
import pyoracle as po

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2005_07547_b200 as pb  # noqa: E402


def _checker(*a):
    return po.RefModelStore(*a) if po.model_ref_available() else po.OracleModelStore(*a)


def _same_dump(g, r):
    eg, wg, ag = g.dump()
    er, wr, ar = r.dump()
    assert len(eg) == len(er) > 0
    for f in po.MODEL_ENTRY_DTYPE.names:
        np.testing.assert_array_equal(np.ascontiguousarray(eg[f]).view(np.uint8),
                                      np.ascontiguousarray(er[f]).view(np.uint8), err_msg=f)
    np.testing.assert_array_equal(wg.view(np.uint64), wr.view(np.uint64))
    np.testing.assert_array_equal(ag.view(np.uint64), ar.view(np.uint64))
    return eg


@pytest.mark.parametrize("res,t_max,min_samples", [(16, 64.0, 32), (5, 2.0, 1), (1, np.inf, 4)])
def test_model_store_bitwise(res, t_max, min_samples):
    rng = np.random.default_rng(res * 31 + min_samples)
    g = pb.ModelStore(res, t_max, min_samples, capacity_log2=12)
    r = _checker(res, t_max, min_samples)
    for frame in range(4):
        k, u, v, c, keys = mc.model_records(rng, 6000, 400)
        perm = rng.permutation(len(k))  # the device sorts: input order is irrelevant
        g.apply(k[perm], u[perm], v[perm], c[perm])
        r.apply(k, u, v, c)
        _same_dump(g, r)
        g.end_frame()
        r.end_frame()
        e = _same_dump(g, r)
    st = g.stats()
    assert st["entries"] == len(e) and st["warm"] == int(e["warm"].sum()) and st["dropped_records"] == 0
    q, u, v = mc.probe_points(rng, keys, 5000)
    ent = g.lookup_warm(q).cpu().numpy()
    pr, found = r.pdf(q, u, v)
    np.testing.assert_array_equal(ent >= 0, found)
    assert found.sum() > 50
    pg = g.pdf(torch.from_numpy(ent), u, v).cpu().numpy()
    np.testing.assert_array_equal(pg.view(np.uint64), pr.view(np.uint64))
    sg = [x.cpu().numpy() for x in g.sample(torch.from_numpy(ent), u, v)]
    sr = r.sample(q, u, v)[:3]
    for a, b in zip(sg, sr):
        np.testing.assert_array_equal(a.view(np.uint64), b.view(np.uint64))


def test_model_lookup_levels():
    """the estimator's coarse-to-fine search (estimators.cpp:464-469): first warm model over
    levels selectLevel(footprint)..maxLevel of keyFor(pos, wo, l) with the Lo store's keys"""
    cfg = po.Config.make(capacity_log2=10, base_cell_size=0.5)
    keyer = pb.FieldStore(pb.FieldStoreConfig(capacity_log2=10, base_cell_size=0.5))
    ok = po.OracleStore(cfg)
    rng = np.random.default_rng(77)
    n = 4000
    pos = rng.uniform(-4, 4, size=(n, 3))
    d = inputs.random_dirs(rng, n)
    fp = np.exp(rng.uniform(np.log(0.01), np.log(20.0), size=n))
    g = pb.ModelStore(8, 64.0, 2, capacity_log2=14)
    r = _checker(8, 64.0, 2)
    # records at levels 0-2 for 30% of the points each: searches stop early, fall back to a
    # coarser level, or find nothing (footprints selecting levels 3-4)
    for l in range(3):
        sel = rng.random(n) < 0.3
        kk = ok.keys_for(pos[sel], d[sel], np.full(int(sel.sum()), l, np.int32))
        kk = np.concatenate([kk] * 3)
        u, v, c = rng.random(len(kk)), rng.random(len(kk)), rng.exponential(1.0, len(kk))
        g.apply(kk, u, v, c)
        r.apply(kk, u, v, c)
    g.end_frame()
    r.end_frame()
    got = g.lookup_warm_levels(keyer, pos, d, fp).cpu().numpy()
    want = np.full(n, -1)
    lv0 = ok.select_levels(fp)
    for l in range(cfg.max_level, -1, -1):
        kk = ok.keys_for(pos, d, np.full(n, l, np.int32))
        ent = g.lookup_warm(kk).cpu().numpy()
        _, found = r.pdf(kk, np.zeros(n), np.zeros(n))
        np.testing.assert_array_equal(ent >= 0, found)
        hit = (l >= lv0) & found
        want[hit] = ent[hit]
    np.testing.assert_array_equal(got, want)
    assert (got >= 0).sum() > 500 and (got < 0).sum() > 100


def test_model_table_full_counts_drops():
    """the device table is bounded (the reference map is not): keys beyond capacity are
    counted, never written over other entries"""
    rng = np.random.default_rng(3)
    g = pb.ModelStore(4, 64.0, 1, capacity_log2=5)
    k, u, v, c, keys = mc.model_records(rng, 3000, 200)
    g.apply(k, u, v, c)
    g.end_frame()
    st = g.stats()
    e, _, _ = g.dump()
    assert st["entries"] == 32 == len(e)
    assert st["dropped_records"] == len(k) - int(e["records"].sum()) > 0
    r = _checker(4, 64.0, 1)
    r.apply(k, u, v, c)
    r.end_frame()
    er, wr, _ = r.dump()
    eg, wg, _ = g.dump()
    idx = {tuple(x["cell"]) + tuple(x["dir"]) + (int(x["level"]),): i for i, x in enumerate(er)}
    for i, x in enumerate(eg):  # every stored entry equals the unbounded reference's
        j = idx[tuple(x["cell"]) + tuple(x["dir"]) + (int(x["level"]),)]
        assert x["records"] == er[j]["records"]
        np.testing.assert_array_equal(wg[i].view(np.uint64), wr[j].view(np.uint64))


def test_model_store_atomic_mode():
    """ATOMIC mode (no sort): entries, counts, warm flags exact; accumulators and weights within
    1e-12 relative of the canonical order."""
    rng = np.random.default_rng(123)
    g = pb.ModelStore(16, 64.0, 8, capacity_log2=12)
    r = _checker(16, 64.0, 8)
    for frame in range(3):
        k, u, v, c, keys = mc.model_records(rng, 20000, 600)
        g.apply(k, u, v, c, mode=pb.MODE_ATOMIC)
        r.apply(k, u, v, c)
        for end in (False, True):
            if end:
                g.end_frame()
                r.end_frame()
            eg, wg, ag = g.dump()
            er, wr, ar = r.dump()
            assert len(eg) == len(er)
            for f in ("level", "cell", "dir", "warm", "c_old", "c_new", "records", "record_count"):
                np.testing.assert_array_equal(eg[f], er[f], err_msg=f)
            np.testing.assert_allclose(eg["total"], er["total"], rtol=1e-12)
            np.testing.assert_allclose(wg, wr, rtol=1e-12, atol=1e-300)
            np.testing.assert_allclose(ag, ar, rtol=1e-12, atol=1e-300)



@pytest.mark.parametrize("leaves,tsplit,t_max", [(64, 4.0, 64.0), (8, 1.5, 3.0), (2, 1.01, np.inf)])
def test_kdtree_model_store_bitwise(leaves, tsplit, t_max):
    """SphericalKdTree kind (models.cpp:96-298, the split-collapse
    learner): node probabilities, accumulators, masses and topology bitwise over frames with a
    hot corner, then lookup, pdf and sample."""
    rng = np.random.default_rng(leaves * 7)
    g = pb.ModelStore(16, t_max, 4, capacity_log2=10, kind=pb.MODEL_KDTREE, kd_leaf_count=leaves,
                      kd_split_threshold=tsplit)
    if po.model_ref_available():
        r = po.RefModelStore(16, t_max, 4, kind=1, leaves=leaves, tsplit=tsplit)
    else:
        r = po.OracleModelStore(16, t_max, 4, kind=1, leaves=leaves, tsplit=tsplit)
    for frame in range(6):
        k, u, v, c, keys = mc.model_records(rng, 5000, 150, skew=3.0)
        perm = rng.permutation(len(k))
        g.apply(k[perm], u[perm], v[perm], c[perm])
        r.apply(k, u, v, c)
        _same_dump(g, r)
        g.end_frame()
        r.end_frame()
        _same_dump(g, r)
        (gi, gf), (ri, rf) = g.dump_tree(), r.dump_tree()
        np.testing.assert_array_equal(gi, ri)
        np.testing.assert_array_equal(gf.view(np.uint64), rf.view(np.uint64))
    q, u, v = mc.probe_points(rng, keys, 3000)
    ent = g.lookup_warm(q).cpu().numpy()
    pr, found = r.pdf(q, u, v)
    np.testing.assert_array_equal(ent >= 0, found)
    assert found.sum() > 50
    pg = g.pdf(torch.from_numpy(ent), u, v).cpu().numpy()
    np.testing.assert_array_equal(pg.view(np.uint64), pr.view(np.uint64))
    sg = [x.cpu().numpy() for x in g.sample(torch.from_numpy(ent), u, v)]
    for a, b in zip(sg, r.sample(q, u, v)[:3]):
        np.testing.assert_array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("comps,alpha,skew,edges", [(4, 0.7, 2.0, True), (3, 0.95, 1.0, False),
                                                   (3, 0.95, 1.0, True), (1, 0.6, 3.0, True)])
def test_gmm_model_store_close(comps, alpha, skew, edges):
    """Gmm kind (models.cpp:427-702, the batch E-step by prefix sums), with
    two apply calls per frame (samples keep call order).  Counters, warm flags, the step index,
    underflows and reseeds are exact.  The state goes through exp/log/pow (not glibc's) and
    differently associated sums: on streams without edge values it agrees to rtol 1e-9
    throughout (weights, means, covariances, statistics, cache, pdf, sample).  Streams with
    border uv / duplicates can leave a hot new entry ill-conditioned: there the statistics,
    weights and means are held to 1e-6 and the inverse-covariance cache is not compared."""
    rng = np.random.default_rng(comps * 13 + int(alpha * 100))
    g = pb.ModelStore(16, 64.0, 4, capacity_log2=10, kind=pb.MODEL_GMM, gmm_components=comps,
                      gmm_alpha_em=alpha)
    if po.model_ref_available():
        r = po.RefModelStore(16, 64.0, 4, kind=2, comps=comps, alpha_em=alpha)
    else:
        r = po.OracleModelStore(16, 64.0, 4, kind=2, comps=comps, alpha_em=alpha)
    C = comps
    tol = 1e-6 if edges else 1e-9
    for frame in range(5):
        k, u, v, c, keys = mc.model_records(rng, 4000, 120, skew=skew)
        if not edges:
            u, v = rng.random(len(k)) ** skew, rng.random(len(k)) ** skew
            c = rng.exponential(1.0, len(k)) + 0.1
        half = len(k) // 2
        for s in (g, r):
            s.apply(k[:half], u[:half], v[:half], c[:half])
            s.apply(k[half:], u[half:], v[half:], c[half:])
            s.end_frame()
        eg, sg, _ = g.dump()
        er, sr, _ = r.dump()
        assert len(eg) == len(er)
        for f in ("level", "cell", "dir", "warm", "c_old", "c_new", "records", "record_count"):
            np.testing.assert_array_equal(eg[f], er[f], err_msg=f)
        np.testing.assert_array_equal(sg[:, 21 * C:], sr[:, 21 * C:])  # i, underflows, reseeds
        upto = 21 * C if not edges else 3 * C  # W, M (+ V, U, cache on clean streams)
        np.testing.assert_allclose(sg[:, :upto], sr[:, :upto], rtol=tol, atol=1e-12)
        np.testing.assert_allclose(sg[:, 6 * C:14 * C], sr[:, 6 * C:14 * C], rtol=tol, atol=1e-12)
    q, u, v = mc.probe_points(rng, keys, 2000)
    us = rng.random(len(q))
    ent = g.lookup_warm(q).cpu().numpy()
    pr, found = r.pdf(q, u, v)
    np.testing.assert_array_equal(ent >= 0, found)
    assert found.sum() > 50
    if edges:
        return
    pg = g.pdf(torch.from_numpy(ent), u, v).cpu().numpy()
    np.testing.assert_allclose(pg, pr, rtol=1e-9)
    sg = [x.cpu().numpy() for x in g.sample(torch.from_numpy(ent), u, v, us)]
    for a, b in zip(sg, r.sample(q, u, v, us)[:3]):
        np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-12)
