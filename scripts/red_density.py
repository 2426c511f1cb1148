"""REDs issued per touched slot per frame (the hot-slot measure) on the config-2 stream at
coarser cell sizes (argv: base multipliers)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_07547_b200 as pb  # noqa: E402

for m in [float(x) for x in sys.argv[1:]] or [1.0, 2.0, 4.0, 8.0]:
    base = math.sqrt(12.0) / 256.0 * m
    gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=22, base_cell_size=base))
          for k in (0, 1, 3)]
    prev = 0
    for it in range(4):
        buf, n = pb.synth_generate(1920, 1080, 4, iteration=it)
        pb.vertex_pass(gs[0], gs[1], gs[2], None, buf, n)
        pb.end_frame_all(gs)
        st = [g.stats() for g in gs]
        reds = st[0]["reds_total"] - prev
        prev = st[0]["reds_total"]
        touched = sum(s["touched_last"] for s in st)
    print(f"base x{m:g}: REDs/frame {reds:.3e}, touched {touched}, REDs per touched slot {reds / max(touched, 1):.1f}")
