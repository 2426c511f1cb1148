"""Twin Lo / Lo\\E stores (csrc/field.cu, pstf_field::twin): created alike and updated only
together, they hold identical occupancy and touch marks, and the tiled vertex kernel then takes
Lo\\E's probes from Lo's.  Against the same passes with the relation disabled (PSTF_NO_TWIN):
occupancy, keys, ages and cOld bitwise, values to 1e-9 (ATOMIC sums), including after the
relation is broken by an update of one store alone."""
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

TWIN_NAME = "k_vertex_pass_tiled<1, VT_MINB, true, false, false, false, tru"  # profile names: 63 chars
EXACT = ("checksum", "level", "cell", "dir", "last_touched")


def _break(gs, how):
    """end the relation: an update, invalidation, restore or endFrame of Lo\\E alone"""
    if how == "apply":
        keys = gs[1].snapshot()[:50]
        k = torch.from_numpy(np.stack([keys["level"], keys["cell"][:, 0], keys["cell"][:, 1],
                                       keys["cell"][:, 2], keys["dir"][:, 0], keys["dir"][:, 1],
                                       keys["checksum"].view(np.int32)], 1).astype(np.int32).copy())
        n = len(keys)
        gs[1].apply(k, torch.ones((3, n), dtype=torch.float64), torch.ones(n, dtype=torch.float64),
                    torch.zeros(n, dtype=torch.uint8), pb.MODE_ATOMIC)
    elif how == "invalidate":
        gs[1].invalidate(((-0.5, 0.0, -0.5), (0.5, 1.0, 0.5)))
    elif how == "restore":
        gs[1].restore(gs[1].snapshot()[:100])
    elif how == "end_frame":
        gs[1].end_frame()


def _run(no_twin, break_at=None, frames=5, evict=2, cap=16, how="apply"):
    if no_twin:
        os.environ["PSTF_NO_TWIN"] = "1"
    try:
        gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=cap,
                                                base_cell_size=inputs.BASE_CORNELL * 2.0,
                                                evict_age_frames=evict))
              for k in (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI)]
        used, out = [], []
        for it in range(frames):
            if it == break_at:
                _break(gs, how)
            buf, n = pb.synth_generate(320, 180, 4, iteration=it)
            pb.profile_enable(True)
            pb.vertex_pass(gs[0], gs[1], gs[2], None, buf, n)
            pb.profile_enable(False)
            used.append(any(TWIN_NAME in k for k in pb.profile_collect()))
            pb.end_frame_all(gs)
            out.append([s.slots() for s in gs])
        return used, out
    finally:
        os.environ.pop("PSTF_NO_TWIN", None)


def _same(a_frames, b_frames):
    for a_it, b_it in zip(a_frames, b_frames):
        for a, b in zip(a_it, b_it):
            gu.assert_slots_bitwise(a, b, EXACT)
            live = b["checksum"] != 0
            np.testing.assert_array_equal(a["c_old"][live], b["c_old"][live])
            np.testing.assert_allclose(a["value_old"][live], b["value_old"][live], rtol=1e-9)


def test_twin_equals_separate_probes():
    used_t, twin = _run(False)
    used_s, sep = _run(True)
    assert all(used_t) and not any(used_s)
    _same(twin, sep)
    for fr in twin:  # the relation's premise: identical occupancy and marks
        gu.assert_slots_bitwise(fr[0], fr[1], EXACT)


@pytest.mark.parametrize("how", ["apply", "invalidate", "restore", "end_frame"])
def test_twin_broken_by_a_single_store_update(how):
    used_t, twin = _run(False, break_at=2, how=how)
    used_s, sep = _run(True, break_at=2, how=how)
    assert used_t == [True, True, False, False, False] and not any(used_s)
    _same(twin, sep)
