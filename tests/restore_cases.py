"""Inputs of the snapshot-restore parity tests, shared by the CPU pin
(tests/test_oracle_pin.py: oracle vs the reference's own insert) and the GPU parity tests."""
import numpy as np

import inputs
import pyoracle as po


def random_updates(store, rng, n, n_keys, levels=3):
    """n counter/accumulate updates over n_keys random keys (1% NaN weights: rejected)."""
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


def restore_records(rng, cap_src=12, n_keys=3000, dup_frac=0.05):
    """Snapshot records of a filled store (values and cOld from real blends), plus duplicate keys
    carrying other values, in shuffled order: the input of a snapshot restore."""
    cfg = po.Config.make(capacity_log2=cap_src, base_cell_size=0.5)
    src = po.OracleStore(cfg)
    for _ in range(2):
        src.queue_apply(random_updates(src, rng, 3 * n_keys, n_keys))
        src.end_frame()
    recs = src.snapshot()
    dup = recs[rng.random(len(recs)) < dup_frac].copy()
    dup["value"] = rng.uniform(0, 3, size=(len(dup), 3))
    dup["c_old"] = rng.uniform(0, 9, size=len(dup))
    allr = np.concatenate([recs, dup])
    return allr[rng.permutation(len(allr))]


def expected_restore(recs):
    """Key-sorted unique records, each key carrying its last record's value (input order)."""
    order = np.lexsort((recs["dir"][:, 1], recs["dir"][:, 0], recs["cell"][:, 2],
                        recs["cell"][:, 1], recs["cell"][:, 0], recs["level"]))  # stable
    s = recs[order]
    k = np.ascontiguousarray(np.column_stack([s["level"], s["cell"], s["dir"]]))
    last = np.ones(len(s), bool)
    last[:-1] = (k[1:] != k[:-1]).any(1)
    return np.ascontiguousarray(s[last])
