"""ORDERED-mode diagnostics on the config-2 stream (run with PSTF_ORDERED_DEBUG=1)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_07547_b200 as pb  # noqa: E402
base = math.sqrt(12.0) / 256.0
gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=22, base_cell_size=base)) for k in (0, 1, 3)]
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    buf, n = pb.synth_generate(1920, 1080, 4, iteration=it)
    pb.vertex_pass(gs[0], gs[1], gs[2], None, buf, n, mode=pb.MODE_ORDERED)
    pb.end_frame_all(gs)
