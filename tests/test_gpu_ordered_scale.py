"""ORDERED mode's slot-grouped fast path (field.cu, fold_slot_records) against the general path
(every value call through the full canonical sort, PSTF_ORDERED_GENERAL) at scale: the config-2
stream (1080p x 4 bounces, 2^22 slots), a coarse-cell stream whose hot slots take tens of
thousands of calls (long runs of equal sort keys, the re-sorted marked runs), and the glossy
scene.  Every slot array, accumulators included, must be bitwise identical frame after frame,
and the fast path must actually have run."""
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import gpu_util as gu  # noqa: E402
import inputs  # noqa: E402
import paper_2005_07547_b200 as pb  # noqa: E402


def _run(general, W, H, B, frames, cap, mult, evict, scene, li=False):
    if general:
        os.environ["PSTF_ORDERED_GENERAL"] = "1"
    try:
        kinds = [pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI] + ([pb.KIND_LI] if li else [])
        gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=cap,
                                                base_cell_size=inputs.BASE_CORNELL * mult,
                                                evict_age_frames=evict))
              for k in kinds]
        out, kernels = [], set()
        for it in range(frames):
            buf, n = pb.synth_generate(W, H, B, iteration=it, scene=scene)
            pb.profile_enable(True)
            pb.vertex_pass(gs[0], gs[1], gs[2], gs[3] if li else None, buf, n,
                           mode=pb.MODE_ORDERED)
            pb.profile_enable(False)
            kernels |= set(pb.profile_collect())
            pb.end_frame_all(gs)
            out.append([s.slots() for s in gs])
        return out, kernels
    finally:
        os.environ.pop("PSTF_ORDERED_GENERAL", None)


def test_ordered_fast_path_equals_general_with_li():
    """config-2 scale with the Li store (a fourth store in the sort key's store field)"""
    fast, kf = _run(False, 1920, 1080, 4, 2, 22, 1.0, 64, 0, li=True)
    gen, _ = _run(True, 1920, 1080, 4, 2, 22, 1.0, 64, 0, li=True)
    assert "k_run_check" in kf
    for it in range(2):
        for a, b in zip(fast[it], gen[it]):
            gu.assert_slots_bitwise(a, b)


@pytest.mark.parametrize("W,H,B,frames,cap,mult,evict,scene,fast_runs", [
    (1920, 1080, 4, 3, 22, 1.0, 64, 0, True),   # config 2
    (640, 360, 4, 4, 18, 4.0, 2, 0, True),      # coarser cells: hot slots, long runs, evictions
    (640, 360, 4, 3, 18, 1.0, 64, 1, True),     # glossy scene
    # very coarse cells: checksum aliases share slots, so the whole pass takes the general path
    (640, 360, 4, 3, 16, 30.0, 2, 0, False),
])
def test_ordered_fast_path_equals_general(W, H, B, frames, cap, mult, evict, scene, fast_runs):
    fast, kf = _run(False, W, H, B, frames, cap, mult, evict, scene)
    gen, kg = _run(True, W, H, B, frames, cap, mult, evict, scene)
    if fast_runs:
        assert "k_slot_fold_long" in kf and "k_run_check" in kf  # the fast path ran
    assert "k_run_check" not in kg
    for it in range(frames):
        for a, b in zip(fast[it], gen[it]):
            gu.assert_slots_bitwise(a, b)


def _run_kernel(perthread, li, W=640, H=360, B=4, frames=4, cap=18):
    if perthread:
        os.environ["PSTF_ORDERED_PERTHREAD"] = "1"
    try:
        ks = [pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI] + ([pb.KIND_LI] if li else [])
        gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=cap,
                                                base_cell_size=inputs.BASE_CORNELL * 2.0,
                                                evict_age_frames=2))
              for k in ks]
        out, kernels = [], set()
        for it in range(frames):
            buf, n = pb.synth_generate(W, H, B, iteration=it)
            pb.profile_enable(True)
            pb.vertex_pass(gs[0], gs[1], gs[2], gs[3] if li else None, buf, n,
                           mode=pb.MODE_ORDERED)
            pb.profile_enable(False)
            kernels |= set(pb.profile_collect())
            pb.end_frame_all(gs)
            out.append([s.slots() for s in gs])
        return out, kernels
    finally:
        os.environ.pop("PSTF_ORDERED_PERTHREAD", None)


@pytest.mark.parametrize("li", [False, True])
def test_ordered_tiled_kernel_equals_per_thread_kernel(li):
    """The ORDERED instantiation of the TMA-tiled vertex kernel (chunk-reserved pairs, holes)
    against the per-thread ORDERED kernel: every slot array bitwise, with and without Li."""
    tiled, kt = _run_kernel(False, li)
    per, kp = _run_kernel(True, li)
    assert any("k_vertex_pass_tiled" in k for k in kt)
    assert not any("k_vertex_pass_tiled" in k for k in kp)
    for a_it, b_it in zip(tiled, per):
        for a, b in zip(a_it, b_it):
            gu.assert_slots_bitwise(a, b)


@pytest.mark.parametrize("W,H,B", [(10, 10, 2), (20, 10, 1), (33, 7, 3), (128, 72, 4)])
def test_ordered_small_passes_equal_per_thread_kernel(W, H, B):
    """Small ORDERED passes through the tiled kernel (a few tiles, most warps reserving a pair
    chunk they barely use) equal the per-thread kernel, frame after frame."""
    tiled, _ = _run_kernel(False, False, W=W, H=H, B=B, frames=3, cap=12)
    per, _ = _run_kernel(True, False, W=W, H=H, B=B, frames=3, cap=12)
    for a_it, b_it in zip(tiled, per):
        for a, b in zip(a_it, b_it):
            gu.assert_slots_bitwise(a, b)


@pytest.mark.parametrize("mode", ["atomic", "ordered"])
def test_empty_passes(mode):
    """n = 0 through the device and the host entry points: no error, nothing changes."""
    gm = pb.MODE_ATOMIC if mode == "atomic" else pb.MODE_ORDERED
    gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=12,
                                            base_cell_size=inputs.BASE_CORNELL))
          for k in (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI)]
    buf, n = pb.synth_generate(16, 8, 2, iteration=0)
    pb.vertex_pass(gs[0], gs[1], gs[2], None, buf, n, mode=gm)
    pb.end_frame_all(gs)
    before = [s.slots() for s in gs]
    pb.vertex_pass(gs[0], gs[1], gs[2], None, buf, 0, mode=gm)
    pb.vertex_pass_host(gs[0], gs[1], gs[2], None, buf.cpu(), 0, mode=gm)
    for s, b in zip(gs, before):
        gu.assert_slots_bitwise(s.slots(), b)
