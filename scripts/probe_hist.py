"""Probe distances of the live slots after the config-2 warm-up (8 iteration streams)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_07547_b200 as pb  # noqa: E402

base = math.sqrt(12.0) / 256.0
gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=22, base_cell_size=base)) for k in (0, 1, 3)]
for it in range(10):
    buf, n = pb.synth_generate(1920, 1080, 4, iteration=it % 8)
    pb.vertex_pass(gs[0], gs[1], gs[2], None, buf, n)
    pb.end_frame_all(gs)
for name, s in zip(("Lo", "LoE", "FLi"), gs):
    h = s.probe_histogram()
    tot = h.sum()
    print(name, "live", int(tot), "share at distance 0..5:", [round(float(x) / tot, 4) for x in h[:6]], ">=6:", round(float(h[6:].sum()) / tot, 5))
