"""Host-side cost of one config-2 step's API calls (vertex_pass + end_frame_all), to see whether
the host keeps ahead of the GPU."""
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
for i in range(16):
    pb.vertex_pass(stores[0], stores[1], stores[2], None, bufs[i % 8], n)
    pb.end_frame_all(stores)
torch.cuda.synchronize()
tv, te, tot = [], [], []
t00 = time.perf_counter()
for i in range(20):
    t0 = time.perf_counter()
    pb.vertex_pass(stores[0], stores[1], stores[2], None, bufs[i % 8], n)
    t1 = time.perf_counter()
    pb.end_frame_all(stores)
    t2 = time.perf_counter()
    tv.append(t1 - t0)
    te.append(t2 - t1)
torch.cuda.synchronize()
print("vertex_pass host us: median %.1f max %.1f" % (sorted(tv)[10] * 1e6, max(tv) * 1e6))
print("end_frame_all host us: median %.1f (includes waiting for the vertex kernel)" % (sorted(te)[10] * 1e6))
print("wall per step ms %.3f" % ((time.perf_counter() - t00) / 20 * 1e3))
pb.profile_collect()
pb.profile_enable(True)
torch.cuda.synchronize()
t00 = time.perf_counter()
for i in range(20):
    pb.vertex_pass(stores[0], stores[1], stores[2], None, bufs[i % 8], n)
    pb.end_frame_all(stores)
torch.cuda.synchronize()
print("with launch events: wall per step ms %.3f" % ((time.perf_counter() - t00) / 20 * 1e3))
pb.profile_enable(False)
