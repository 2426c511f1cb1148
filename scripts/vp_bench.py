"""Quick per-kernel timing of one config-2 iteration (used while optimising; not the bench)."""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2005_07547_b200 as pb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=6)
p.add_argument("--warmup", type=int, default=3)
p.add_argument("--streams", type=int, default=3)
p.add_argument("--width", type=int, default=1920)
p.add_argument("--height", type=int, default=1080)
p.add_argument("--bounces", type=int, default=4)
p.add_argument("--cap", type=int, default=22)
p.add_argument("--base-mult", type=float, default=1.0, help="cell size multiplier (coarser cells: hotter slots)")
args = p.parse_args()

base = math.sqrt(12.0) / 256.0 * args.base_mult
stores = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=args.cap, base_cell_size=base))
          for k in (0, 1, 3)]
bufs = []
for i in range(args.streams):
    b, n = pb.synth_generate(args.width, args.height, args.bounces, iteration=i)
    bufs.append(b)
for i in range(args.warmup):
    pb.vertex_pass(stores[0], stores[1], stores[2], None, bufs[i % len(bufs)], n)
    pb.end_frame_all(stores)
torch.cuda.synchronize()
pb.profile_collect()
pb.profile_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(args.steps):
    pb.vertex_pass(stores[0], stores[1], stores[2], None, bufs[i % len(bufs)], n)
    pb.end_frame_all(stores)
e1.record()
torch.cuda.synchronize()
pb.profile_enable(False)
prof = pb.profile_collect()
ms = e0.elapsed_time(e1) / args.steps
print(f"step {ms:.3f} ms  -> {n / ms / 1e6:.3f} G vertices/s")
for k, (t, c) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:40s} {t / args.steps:8.4f} ms/step  launches {c}")
print("stats", [s.stats() for s in stores])
