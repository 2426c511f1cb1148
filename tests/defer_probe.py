"""Helper for test_gpu_parity.test_deferred_phase2_identical: a short vertex-pass sequence
(new keys every frame, queries and stats between passes) whose slot arrays and query results are
written to an .npz; run once with and once without PSTF_NO_DEFER."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))
import numpy as np  # noqa: E402

import inputs  # noqa: E402
import paper_2005_07547_b200 as pb  # noqa: E402

out = sys.argv[1]
cfg = lambda k: pb.FieldStoreConfig(kind=k, capacity_log2=13, base_cell_size=inputs.BASE_CORNELL * 3)
st = [pb.FieldStore(cfg(k)) for k in (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI)]
res = {}
for it in range(5):
    buf, n = pb.synth_generate(64, 36, 4, iteration=it, cam_shift_x=0.05 * it)
    pb.vertex_pass(st[0], st[1], st[2], None, buf, n)
    if it % 2:
        res[f"stats{it}"] = np.array([list(s.stats().values()) for s in st], np.int64)
    if it == 3:
        pb.vertex_pass(st[0], st[1], st[2], None, buf, n)  # two passes in one frame
    if it == 2:
        st[2].end_frame()  # a single store's endFrame while the pass is pending
        st[0].end_frame()
        st[1].end_frame()
    else:
        pb.end_frame_all(st)
for i, s in enumerate(st):
    res[f"slots{i}"] = np.ascontiguousarray(s.slots()).view(np.uint8)
np.savez(out, **res)
