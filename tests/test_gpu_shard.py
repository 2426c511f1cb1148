"""Key-owner sharding on the GPU library, emulated in one process on one device: `world`
independent replicas (separate stores) driven in lock-step through the CudaBackend operations,
with the collectives done in-process between the phases (no kernel ever waits on another rank).
The result must equal the unsharded single-GPU vertex pass: occupancy, keys, ages and c_old
exactly, values to 1e-9; all replicas identical."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import gpu_util as gu  # noqa: E402
import inputs  # noqa: E402
import paper_2005_07547_b200 as pb  # noqa: E402
from paper_2005_07547_b200.shard import (DELTA_BYTES, PARTIAL_BYTES, CudaBackend)  # noqa: E402


def _stores(cap, base, evict):
    return [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=cap, base_cell_size=base,
                                              evict_age_frames=evict))
            for k in (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI)]


@pytest.mark.parametrize("world,cap,mult,evict,counted", [(2, 12, 8.0, 2, False),
                                                          (4, 14, 1.0, 64, False),
                                                          (2, 10, 30.0, 2, False),
                                                          (2, 12, 8.0, 2, True),
                                                          (4, 14, 1.0, 64, True)])
def test_sharded_emulation_equals_single_gpu(world, cap, mult, evict, counted):
    """counted: the exchanges whose sizes stay on the device (pstf_pending_count_dev,
    pstf_partials_export_async, pstf_end_frame_commit_async), as ShardedFieldCache uses them
    over NCCL"""
    W, H, B, frames = 96, 54, 4, 4
    base = inputs.BASE_CORNELL * mult
    single = _stores(cap, base, evict)
    reps = [_stores(cap, base, evict) for _ in range(world)]
    bes = [CudaBackend(r, rank, world) for rank, r in enumerate(reps)]
    n_paths = W * H
    for it in range(frames):
        buf, n = pb.synth_generate(W, H, B, iteration=it)
        pb.vertex_pass(single[0], single[1], single[2], None, buf, n)
        pb.end_frame_all(single)
        # 1: local pass per rank on its stripe
        for r, be in enumerate(bes):
            p0, p1 = n_paths * r // world, n_paths * (r + 1) // world
            sb, sn = pb.synth_generate(W, H, B, iteration=it, path0=p0, npaths=p1 - p0)
            be.vertex_pass_local((sb, sn))
        # 2: all-gather pending records, identical placement everywhere
        if counted:
            allrec = torch.cat([be.pending_bytes_n(int(be.pending_count_dev().item()))
                                for be in bes])
        else:
            allrec = torch.cat([be.pending_bytes() for be in bes])
        for be in bes:
            be.resolve(allrec)
        # 3: partials to owners (all-to-all)
        if counted:
            outs = []
            for be in bes:
                buf_s, cnt = be.partials_export_async()
                outs.append((buf_s, [int(x) for x in cnt.tolist()]))
        else:
            outs = [be.partials_export() for be in bes]
        for r, be in enumerate(bes):
            parts = []
            for src, (buf_s, counts) in enumerate(outs):
                off = sum(counts[:r]) * PARTIAL_BYTES
                parts.append(buf_s[off:off + counts[r] * PARTIAL_BYTES])
            be.partials_import(torch.cat(parts))
        # 4: global pass-1 sums
        sums = sum(be.end_frame_reduce() for be in bes)
        # 5: commit + all-gather deltas
        if counted:
            parts = [be.end_frame_commit_async(sums) for be in bes]
            deltas = torch.cat([buf[:int(nd.item())] for buf, nd in parts])
        else:
            deltas = torch.cat([be.end_frame_commit(sums) for be in bes])
        for be in bes:
            be.deltas_import(deltas)
        torch.cuda.synchronize()
        for s in range(3):
            want = single[s].slots()
            for r in range(world):
                got = reps[r][s].slots()
                gu.assert_slots_bitwise(got, want, ("checksum", "level", "cell", "dir",
                                                    "last_touched"))
                live = want["checksum"] != 0
                np.testing.assert_array_equal(got["c_old"][live], want["c_old"][live])
                np.testing.assert_allclose(got["value_old"][live], want["value_old"][live],
                                           rtol=1e-9)
                assert reps[r][s].stats()["live"] == single[s].stats()["live"]
            assert sum(reps[r][s].stats()["dropped"] for r in range(world)) == \
                single[s].stats()["dropped"]
