"""Phase-2 (new-key placement) cost of a filling step: kernel times + host wall time."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2005_07547_b200 as pb  # noqa: E402

base = math.sqrt(12.0) / 256.0
stores = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=22, base_cell_size=base)) for k in (0, 1, 3)]
bufs = [pb.synth_generate(1920, 1080, 4, iteration=i)[0] for i in range(8)]
n = 1920 * 1080 * 4
for i in range(3):
    pb.vertex_pass(stores[0], stores[1], stores[2], None, bufs[i], n)
    pb.end_frame_all(stores)
torch.cuda.synchronize()
for i in range(3, 7):
    pb.profile_collect()
    pb.profile_enable(True)
    t0 = time.perf_counter()
    pb.vertex_pass(stores[0], stores[1], stores[2], None, bufs[i], n)
    pb.end_frame_all(stores)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pb.profile_enable(False)
    prof = pb.profile_collect()
    st = [s.stats() for s in stores]
    ktot = sum(v[0] for v in prof.values())
    print(f"step {i}: wall {1e3 * (t1 - t0):.3f} ms kernels {ktot:.3f} ms new {[x['new_keys_last'] for x in st]} rounds {st[0]['placement_rounds_last']}")
    for k, (t, c) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        print(f"   {k[:60]:60s} {t:.4f} ms x{c}")
