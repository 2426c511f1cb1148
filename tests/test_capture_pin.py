"""Pins the captured-stream path (oracle/_ref/libpstf_capture.so) on CPU: the reference path
tracer's VertexRecords, converted to the canonical SoA record and replayed through the restated
onVertex (oracle/ref_shim.cpp over the reference FieldStore, and the C oracle), leave the field
stores byte-identical to the reference's own EstimatorRun(PT_NEE, deterministic) rendering the
same frames (estimators.cpp:560-655) — so a GPU replay of a captured stream that matches the
replay matches the reference renderer itself (SURVEY.md Appendix B probe 3)."""
import numpy as np
import pytest

import pyoracle as po

pc = pytest.importorskip("pycapture")
if not pc.available() or not po.ref_available():  # pragma: no cover
    pytest.skip("oracle/_ref capture/reference libraries not built", allow_module_level=True)


@pytest.mark.parametrize("scene,size,frames,li,masks", [
    ("cornell.scene", 48, 3, False, (7, 7)),
    ("staircase_glossy.scene", 40, 3, True, (2, 5)),
    ("furnace_env.scene", 32, 3, True, (7, 3)),
])
def test_capture_replay_equals_estimator_run(scene, size, frames, li, masks):
    sc = pc.Scene(scene, size, size)
    run = pc.RefEstimatorRun(sc, kind=pc.PT_NEE, deterministic=True, capacity_log2=14,
                             track_li=li, loe_mask=masks[0], fli_mask=masks[1])
    cfg = run.store_config(0)
    kinds = (po.KIND_LO, po.KIND_LOE, po.KIND_FLI) + ((po.KIND_LI,) if li else ())
    mk = lambda cls: [cls(po.Config.make(kind=k, capacity_log2=14,
                                         base_cell_size=cfg["base_cell_size"])) for k in kinds]
    ref, orc = mk(po.RefStore), mk(po.OracleStore)
    escapes = 0
    for f in range(frames):
        buf, n, depth = pc.capture_frame(sc, f, seed=0, with_depth=True)
        fl = buf[34 * n:].view(np.uint32)[:n]
        escapes += int((((fl & 1) != 0) & ((fl & 2) == 0)).sum())
        assert depth.min() >= 1
        for st, replay in ((ref, po.vertex_pass_ref), (orc, po.vertex_pass_oracle)):
            replay(st[0], st[1], st[2], st[3] if li else None, buf, n, masks[0], masks[1],
                   deterministic=True)
            for s in st:
                s.end_frame()
        run.frame()
        for w in range(len(kinds)):
            want = run.slots(w).tobytes()
            assert ref[w].slots().tobytes() == want, (f, w)
            assert orc[w].slots().tobytes() == want, (f, w)
    if scene == "furnace_env.scene":
        assert escapes > 0
