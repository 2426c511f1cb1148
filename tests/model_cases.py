"""Record streams for the model-store parity tests: ModelStore<DirGrid>
records (key, uv, contribution) as FieldRecorder::onVertex emits them (estimators.cpp:262-292),
plus the edges the store must handle: uv on the grid borders (0, -0.0, 1.0), zero / negative /
infinite / NaN contributions (rejected by DirGrid::record but counted by applyRecord), exact
duplicate (key, uv) records, and a few very hot keys."""
import numpy as np

import inputs
import pyoracle as po


def model_records(rng, n, n_keys, base=0.5, levels=3, skew=1.0):
    ks = po.OracleStore(po.Config.make(capacity_log2=10, base_cell_size=base))
    pos = rng.uniform(-4, 4, size=(n_keys, 3))
    dirs = inputs.random_dirs(rng, n_keys)
    lv = rng.integers(0, levels, size=n_keys).astype(np.int32)
    keys = ks.keys_for(pos, dirs, lv)
    idx = np.minimum((rng.pareto(1.1, n) * 3).astype(np.int64), n_keys - 1)  # hot keys first
    idx = rng.permutation(n_keys)[idx]
    k = keys[idx]
    u, v = rng.random(n) ** skew, rng.random(n) ** skew  # skew > 1: hot corner (k-d splits)
    c = rng.exponential(1.0, n)
    e = rng.random(n)
    u[e < 0.02] = 1.0
    v[(e >= 0.02) & (e < 0.04)] = 1.0
    u[(e >= 0.04) & (e < 0.05)] = 0.0
    u[(e >= 0.05) & (e < 0.06)] = -0.0
    f = rng.random(n)
    c[f < 0.03] = 0.0
    c[(f >= 0.03) & (f < 0.04)] = -0.5
    c[(f >= 0.04) & (f < 0.045)] = np.inf
    # NaN only where (key, uv) is unique (random uv): std::sort over NaN is otherwise unordered
    c[(f >= 0.045) & (f < 0.05) & (e >= 0.06)] = np.nan
    dup = rng.random(n) < 0.02
    src = rng.integers(0, n, size=int(dup.sum()))
    ok = np.isfinite(c[src])
    src = src[ok]
    k = np.concatenate([k, k[src]])
    u = np.concatenate([u, u[src]])
    v = np.concatenate([v, v[src]])
    c = np.concatenate([c, rng.exponential(1.0, len(src))])
    p = rng.permutation(len(k))
    return k[p], u[p], v[p], c[p], keys


def probe_points(rng, keys, n):
    """query keys (known keys plus a few never recorded) and uv / sample inputs"""
    q = keys[rng.integers(0, len(keys), size=n)].copy()
    q["cell"][: n // 20, 0] += 1000  # unknown keys
    u, v = rng.random(n), rng.random(n)
    u[:5] = [0.0, 1.0, 0.999999, 0.5, 1e-300]
    v[:5] = [1.0, 0.0, 0.999999, 0.5, 1e-300]
    return q, u, v
