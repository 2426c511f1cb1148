"""Multi-rank protocol of the field cache (paper_2005_07547_b200.shard) on CPU: world size 2
(and 4) over gloo with the numpy reference backend (tests/shard_cpu_backend.py): each rank runs
phase 1 on its image stripe, the ranks place the union of new keys identically, all-reduce the
live slots' accumulators and run endFrame.  After several frames every rank's replica must be
identical, and equal to the single-process reference semantics (the C restatement's
deterministic onVertex over the whole frame): occupancy, keys, ages and c_old exactly, values to
1e-9 (summation order differs)."""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
W, H, B, FRAMES = 24, 16, 4, 4


def _cfgs(cap, evict):
    sys.path[:0] = [HERE, os.path.join(HERE, "..", "oracle")]
    import inputs
    import pyoracle as po
    base = inputs.BASE_CORNELL * 8.0
    return [po.Config.make(kind=k, capacity_log2=cap, base_cell_size=base, evict_age_frames=evict)
            for k in (po.KIND_LO, po.KIND_LOE, po.KIND_FLI)]


def _stripe(buf, n_paths, rank, world, po):
    f64, flags = po.soa_views(buf, n_paths * B)
    p0, p1 = n_paths * rank // world, n_paths * (rank + 1) // world
    idx = np.concatenate([np.arange(b * n_paths + p0, b * n_paths + p1) for b in range(B)])
    m = len(idx)
    out = np.zeros(34 * m + (m + 1) // 2, np.float64)
    out[:34 * m] = f64[:, idx].reshape(-1)
    out[34 * m:].view(np.uint32)[:m] = flags[idx]
    return out, m


def _worker(rank, world, port, cap, evict, outdir):
    sys.path[:0] = [HERE, os.path.join(HERE, ".."), os.path.join(HERE, "..", "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import pyoracle as po
    from paper_2005_07547_b200.shard import Collectives, ShardedFieldCache
    from shard_cpu_backend import CpuBackend
    be = CpuBackend(_cfgs(cap, evict), rank, world)
    cache = ShardedFieldCache(be, Collectives(dist, "cpu"))
    for it in range(FRAMES):
        buf, _ = po.synth_generate(W, H, B, iteration=it)
        cache.iteration(_stripe(buf, W * H, rank, world, po))
    np.savez(os.path.join(outdir, f"rank{rank}.npz"),
             **{f"{f}{s}": getattr(r, f) for s, r in enumerate(be.reps)
                for f in ("chk", "lastb", "com", "keyf")},
             live=np.array([r.live for r in be.reps]),
             dropped=np.array([r.dropped for r in be.reps]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,cap,evict", [(2, 9, 2), (2, 12, 64), (4, 10, 2), (2, 9, 0)])
def test_sharded_protocol_matches_single_rank_semantics(tmp_path, world, cap, evict):
    mp.spawn(_worker, args=(world, _free_port(), cap, evict, str(tmp_path)), nprocs=world,
             join=True)
    sys.path[:0] = [os.path.join(HERE, "..", "oracle")]
    import pyoracle as po
    ref = [po.OracleStore(c) for c in _cfgs(cap, evict)] + [None]
    for it in range(FRAMES):
        buf, n = po.synth_generate(W, H, B, iteration=it)
        po.vertex_pass_oracle(*ref, buf, n, deterministic=True)
        for s in ref[:3]:
            s.end_frame()
    res = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    for s in range(3):
        for r in range(1, world):  # replicas converge
            for f in ("chk", "lastb", "keyf"):
                np.testing.assert_array_equal(res[r][f"{f}{s}"], res[0][f"{f}{s}"])
            np.testing.assert_array_equal(res[r][f"com{s}"], res[0][f"com{s}"])
        sl = ref[s].slots()
        got = res[0]
        np.testing.assert_array_equal(got[f"chk{s}"], sl["checksum"])
        live = sl["checksum"] != 0
        np.testing.assert_array_equal((got[f"lastb{s}"].astype(np.int64) - 1)[live],
                                      sl["last_touched"][live])
        np.testing.assert_array_equal(got[f"com{s}"][live, 3], sl["c_old"][live])
        np.testing.assert_allclose(got[f"com{s}"][live, :3], sl["value_old"][live], rtol=1e-9)
        assert got["live"][s] == ref[s].stats()["live"]
        assert sum(rr["dropped"][s] for rr in res) == ref[s].stats()["dropped"]


def _gather_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path[:0] = [os.path.join(HERE, "..")]
    from paper_2005_07547_b200.shard import Collectives
    c = Collectives(dist, "cpu")
    info = c.all_gather_vec(torch.tensor([rank * 10 + 1, 7, rank], dtype=torch.int64))
    sizes = [64 * (r + 1) if r != 1 else 0 for r in range(world)]  # unequal, one empty
    payload = (torch.arange(sizes[rank], dtype=torch.int64) % 251 + rank).to(torch.uint8)
    got = c.gather_known(payload, sizes)
    x = torch.full((5,), float(rank + 1), dtype=torch.float64)
    c.all_reduce_sum(x)
    torch.save({"info": info, "got": got, "sum": x}, os.path.join(outdir, f"g{rank}.pt"))
    dist.destroy_process_group()


def test_collectives_gloo(tmp_path):
    """the protocol's collectives over gloo with CPU tensors: the small-vector all-gather that
    carries the frame's one host read, the known-size byte all-gather (rank order, unequal and
    empty contributions) and the in-place all-reduce"""
    world = 3
    mp.spawn(_gather_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    want = torch.cat([(torch.arange(64 * (r + 1) if r != 1 else 0, dtype=torch.int64) % 251 + r)
                      .to(torch.uint8) for r in range(world)])
    for r in range(world):
        d = torch.load(os.path.join(tmp_path, f"g{r}.pt"))
        assert d["info"] == [[q * 10 + 1, 7, q] for q in range(world)]
        assert torch.equal(d["got"], want)
        assert torch.equal(d["sum"], torch.full((5,), 6.0, dtype=torch.float64))
