"""Per-step new keys / placement rounds of the config-2 loop (how often phase 2 runs and how big)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_07547_b200 as pb  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
base = math.sqrt(12.0) / 256.0
stores = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=22, base_cell_size=base)) for k in (0, 1, 3)]
bufs = []
for i in range(S):
    b, n = pb.synth_generate(1920, 1080, 4, iteration=i)
    bufs.append(b)
for i in range(3 * S):
    pb.vertex_pass(stores[0], stores[1], stores[2], None, bufs[i % S], n)
    st = [s.stats() for s in stores]
    pb.end_frame_all(stores)
    print(i, "new", [x["new_keys_last"] for x in st], "rounds", [x["placement_rounds_last"] for x in st],
          "live", [x["live"] for x in st], "dropped", [x["dropped"] for x in st])
