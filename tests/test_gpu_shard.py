"""The multi-GPU protocol on the GPU library, emulated in one process on one device: `world`
independent replicas (separate stores) driven in lock-step through the CudaBackend operations,
with the collectives done in-process between the phases (no kernel ever waits on another rank).
The result must equal the unsharded single-GPU vertex pass: occupancy, keys, ages and c_old
exactly, values to 1e-9; all replicas bitwise identical."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import gpu_util as gu  # noqa: E402
import inputs  # noqa: E402
import paper_2005_07547_b200 as pb  # noqa: E402
from paper_2005_07547_b200.shard import PENDING_BYTES, CudaBackend  # noqa: E402


def _stores(cap, base, evict):
    return [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=cap, base_cell_size=base,
                                              evict_age_frames=evict))
            for k in (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI)]


@pytest.mark.parametrize("world,cap,mult,evict", [(2, 12, 8.0, 2), (4, 14, 1.0, 64),
                                                  (2, 10, 30.0, 2), (3, 12, 4.0, 3),
                                                  (2, 12, 8.0, 0)])
def test_sharded_emulation_equals_single_gpu(world, cap, mult, evict):
    W, H, B, frames = 96, 54, 4, 5
    base = inputs.BASE_CORNELL * mult
    single = _stores(cap, base, evict)
    reps = [_stores(cap, base, evict) for _ in range(world)]
    bes = [CudaBackend(r, rank, world) for rank, r in enumerate(reps)]
    n_paths = W * H
    for it in range(frames):
        buf, n = pb.synth_generate(W, H, B, iteration=it)
        pb.vertex_pass(single[0], single[1], single[2], None, buf, n)
        pb.end_frame_all(single)
        # 1: phase 1 per rank on its stripe
        for r, be in enumerate(bes):
            p0, p1 = n_paths * r // world, n_paths * (r + 1) // world
            sb, sn = pb.synth_generate(W, H, B, iteration=it, path0=p0, npaths=p1 - p0)
            be.vertex_pass_local((sb, sn))
        # 2: the size vectors (all-gather), pending records (all-gather), identical placement
        info = [be.sync_vector().tolist() for be in bes]
        assert all(i[1] == info[0][1] for i in info) and not any(i[2] for i in info)
        allrec = torch.cat([be.pending_bytes_n(i[0] * PENDING_BYTES) for be, i in zip(bes, info)])
        for be in bes:
            be.resolve(allrec)
        # 3: pack the live slots' accumulators, all-reduce (sum in rank order), unpack
        bound = info[0][1] + sum(i[0] for i in info)
        packs = [be.pack(bound).clone() for be in bes]
        total = packs[0].clone()
        for p in packs[1:]:
            total += p
        # 4: endFrame everywhere (rank 0 through unpack + the ordinary endFrame, the others
        # straight from the packed sums; both must give the same replica)
        for r, be in enumerate(bes):
            if r == 0:
                be.unpack(total)
                be.end_frame()
            else:
                be.commit(total)
        torch.cuda.synchronize()
        for s in range(3):
            want = single[s].slots()
            ref0 = reps[0][s].slots()
            for r in range(world):
                got = reps[r][s].slots()
                gu.assert_slots_bitwise(got, want, ("checksum", "level", "cell", "dir",
                                                    "last_touched"))
                gu.assert_slots_bitwise(got, ref0)  # replicas identical
                live = want["checksum"] != 0
                np.testing.assert_array_equal(got["c_old"][live], want["c_old"][live])
                np.testing.assert_allclose(got["value_old"][live], want["value_old"][live],
                                           rtol=1e-9)
                assert reps[r][s].stats()["live"] == single[s].stats()["live"]
            assert sum(reps[r][s].stats()["dropped"] for r in range(world)) == \
                single[s].stats()["dropped"]
