"""Regenerates the golden fixtures in tests/golden/ from the UNMODIFIED reference field engine
(oracle/_ref/libpstf_ref.so, compiled in place from /root/reference by oracle/Makefile).

  python tests/golden/make_golden.py

Fixtures (all small, np.savez_compressed):
  keys.npz     pos/dir/level inputs and the reference keyFor output at two configs
  levels.npz   footprints and the reference selectLevel output
  vertex.npz   the reference slot arrays after each of 3 frames of a 48x27x4 synthetic stream
               replayed through the public FieldStore API in deterministic mode (EstimatorRun
               deterministic semantics), for Lo/LoE/FLi/Li at 2^11 slots (drops + eviction)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.join(HERE, ".."), os.path.join(HERE, "..", "..", "oracle")]

import inputs  # noqa: E402
import pyoracle as po  # noqa: E402

CONFIGS = {"half": dict(base_cell_size=0.5), "cornell": dict(base_cell_size=inputs.BASE_CORNELL)}
VERTEX = dict(width=48, height=27, bounces=4, frames=3, cap=11, mult=8.0, evict=2)


def main():
    assert po.ref_available(), "build oracle/_ref first (make -C oracle)"
    rng = np.random.default_rng(20260101)
    d = np.concatenate([inputs.random_dirs(rng, 6000), inputs.boundary_dirs(rng, 6000),
                        inputs.structured_dirs(), inputs.special_dirs()])
    n = len(d)
    pos = np.concatenate([inputs.random_positions(rng, n - 8), inputs.special_positions()])
    lv = rng.integers(0, 5, size=n).astype(np.int32)
    out = {"pos": pos, "dir": d, "level": lv}
    for name, kw in CONFIGS.items():
        r = po.RefStore(po.Config.make(capacity_log2=8, **kw))
        k = r.keys_for(pos, d, lv)
        out[f"{name}_keys"] = np.ascontiguousarray(k).view(np.int32).reshape(n, 7)
        out[f"{name}_base"] = np.array(kw["base_cell_size"])
    np.savez_compressed(os.path.join(HERE, "keys.npz"), **out)

    fp = np.concatenate([inputs.level_footprints(inputs.BASE_CORNELL, max_exp=10),
                         inputs.random_footprints(rng, 4000, inputs.BASE_CORNELL)])
    r = po.RefStore(po.Config.make(capacity_log2=8, base_cell_size=inputs.BASE_CORNELL,
                                   max_level=8))
    np.savez_compressed(os.path.join(HERE, "levels.npz"), footprint=fp,
                        level=r.select_levels(fp), base=np.array(inputs.BASE_CORNELL),
                        max_level=np.array(8))

    v = VERTEX
    base = inputs.BASE_CORNELL * v["mult"]
    kinds = (po.KIND_LO, po.KIND_LOE, po.KIND_FLI, po.KIND_LI)
    stores = [po.RefStore(po.Config.make(kind=k, capacity_log2=v["cap"], base_cell_size=base,
                                         evict_age_frames=v["evict"])) for k in kinds]
    vout = {"base": np.array(base)}
    for k, val in v.items():
        vout[k] = np.array(val)
    for it in range(v["frames"]):
        buf, n = po.synth_generate(v["width"], v["height"], v["bounces"], iteration=it)
        po.vertex_pass_ref(*stores, buf, n, deterministic=True, threads=2)
        for si, s in enumerate(stores):
            s.end_frame()
            sl = s.slots()
            vout[f"f{it}_s{si}_slots"] = np.frombuffer(sl.tobytes(), np.uint8)
            st = s.stats()
            vout[f"f{it}_s{si}_stats"] = np.array([st[x] for x in ("frame", "rejected", "dropped",
                                                                   "internal_errors", "live")])
    np.savez_compressed(os.path.join(HERE, "vertex.npz"), **vout)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
