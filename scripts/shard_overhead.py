"""Fixed cost of the key-owner-sharded iteration (paper_2005_07547_b200.shard) on one GPU: a
world-size-1 NCCL group runs the whole protocol (collectives degenerate to copies), compared
with the plain single-GPU step.  Upper bound on what the protocol adds per rank besides the
data exchange itself."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2005_07547_b200 as pb  # noqa: E402
from paper_2005_07547_b200.shard import Collectives, CudaBackend, ShardedFieldCache  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
base = math.sqrt(12.0) / 256.0
n = 1920 * 1080 * 4
bufs = [pb.synth_generate(1920, 1080, 4, iteration=i)[0] for i in range(8)]


def stores():
    return [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=22, base_cell_size=base)) for k in (0, 1, 3)]


def timed(step, k=12):
    for i in range(8):
        step(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(k):
        step(8 + i)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3


s1 = stores()
plain = timed(lambda i: (pb.vertex_pass(s1[0], s1[1], s1[2], None, bufs[i % 8], n), pb.end_frame_all(s1)))
s2 = stores()
sh = ShardedFieldCache(CudaBackend(s2, 0, 1), Collectives(dist, torch.device("cuda", 0)))
shard = timed(lambda i: sh.iteration((bufs[i % 8], n)))
print(f"plain step {plain:.3f} ms, sharded protocol at world 1 {shard:.3f} ms")


# per-step breakdown of the protocol (synchronised timers; world 1)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0)) if not dist.is_initialized() else None
b, c = sh.b, sh.c
acc = {}


def t(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    acc[name] = acc.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return r


K = 8
for i in range(K):
    t("vertex_pass_local", lambda: b.vertex_pass_local((bufs[i % 8], n)))
    recs = t("pending+allgather", lambda: c.all_gather_bytes(b.pending_bytes()))
    t("resolve", lambda: b.resolve(recs))
    out, counts = t("partials_export", lambda: b.partials_export())
    recv = t("all_to_all", lambda: c.all_to_all_bytes(out, counts, 40)[0])
    t("partials_import", lambda: b.partials_import(recv))
    sums = t("ef_reduce+allreduce", lambda: c.all_reduce_sum(b.end_frame_reduce()))
    deltas = t("ef_commit", lambda: b.end_frame_commit(sums))
    g = t("deltas_allgather", lambda: c.all_gather_bytes(deltas))
    t("deltas_import", lambda: b.deltas_import(g))
for k, v in acc.items():
    print(f"  {k:22s} {v / K:.3f} ms")
dist.destroy_process_group()
