"""Fixed cost of the multi-GPU iteration (paper_2005_07547_b200.shard) on one GPU: a world-size-1
NCCL group runs the whole protocol (collectives degenerate to copies), compared with the plain
single-GPU step, plus a synchronised per-phase breakdown and the bytes each collective moves
(the inputs of the N-GPU projection in DESIGN.md section 6)."""
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
from paper_2005_07547_b200.shard import PENDING_BYTES  # noqa: E402
for i in range(K):
    t("vertex_pass_local", lambda: b.vertex_pass_local((bufs[i % 8], n)))
    info = t("sync (all_gather_vec + host read)", lambda: c.all_gather_vec(b.sync_vector()))
    pend = [int(r[0]) for r in info]
    recs = t("pending all_gather", lambda: c.gather_known(b.pending_bytes_n(pend[0] * PENDING_BYTES),
                                                          [p * PENDING_BYTES for p in pend]))
    t("resolve", lambda: b.resolve(recs))
    bound = int(info[0][1]) + sum(pend)
    packed = t("live pack", lambda: b.pack(bound))
    t("all_reduce", lambda: c.all_reduce_sum(packed))
    t("end_frame from the packed sums", lambda: b.commit(packed))
print(f"  live slots packed per frame {bound}, all-reduce payload {bound * 32 / 1e6:.1f} MB")
for k, v in acc.items():
    print(f"  {k:22s} {v / K:.3f} ms")
dist.destroy_process_group()
