"""Hot-slot variant of the tiled vertex kernel (warp aggregation of same-slot REDs,
csrc/field.cu vertex_body<..., AGG>): chosen per launch when the previous frame issued more
than 1000 REDs per touched slot (profiles/round2_match_any_ab.md).  It must give the same
occupancy, keys, ages and cOld as the plain kernel, values within 1e-9, and be selected on
coarse cells only."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import gpu_util as gu  # noqa: E402
import inputs  # noqa: E402
import paper_2005_07547_b200 as pb  # noqa: E402

AGG_NAME = "k_vertex_pass_tiled<1, VT_MINB, true, false, false, true>"


def _run(mult, force=None, frames=6):
    if force is not None:
        os.environ["PSTF_RED_AGG"] = str(force)
    try:
        gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=18,
                                                base_cell_size=inputs.BASE_CORNELL * mult))
              for k in (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI)]
        used, out = [], []
        for it in range(frames):
            buf, n = pb.synth_generate(640, 360, 4, iteration=it)
            pb.profile_enable(True)
            pb.vertex_pass(gs[0], gs[1], gs[2], None, buf, n)
            pb.profile_enable(False)
            used.append(any(AGG_NAME in k for k in pb.profile_collect()))
            pb.end_frame_all(gs)
            # the measure comes back asynchronously; a pass that finds it not yet written keeps
            # the previous choice for one more frame, so let it land before the next pass
            torch.cuda.synchronize()
            out.append([s.slots() for s in gs])
        return used, out
    finally:
        os.environ.pop("PSTF_RED_AGG", None)


def test_agg_kernel_equals_plain_kernel():
    used_a, agg = _run(8.0, force=1)
    used_p, plain = _run(8.0, force=0)
    assert all(used_a) and not any(used_p)
    for a_it, p_it in zip(agg, plain):
        for a, p in zip(a_it, p_it):
            gu.assert_slots_bitwise(a, p, ("checksum", "level", "cell", "dir", "last_touched"))
            live = p["checksum"] != 0
            np.testing.assert_array_equal(a["c_old"][live], p["c_old"][live])
            np.testing.assert_allclose(a["value_old"][live], p["value_old"][live], rtol=1e-9)


def test_agg_selected_on_coarse_cells_only():
    used_coarse, _ = _run(16.0)
    used_fine, _ = _run(1.0)
    # frame 0 inserts every key (no REDs): measured again at frame 1, used from frame 2 on
    assert not used_coarse[0] and all(used_coarse[2:])
    assert not any(used_fine)
