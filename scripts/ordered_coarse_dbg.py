import sys; sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo')
import paper_2005_07547_b200 as pb, inputs
gs = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=16, base_cell_size=inputs.BASE_CORNELL * 30, evict_age_frames=2)) for k in (0, 1, 3)]
for it in range(3):
    buf, n = pb.synth_generate(640, 360, 4, iteration=it)
    pb.vertex_pass(gs[0], gs[1], gs[2], None, buf, n, mode=pb.MODE_ORDERED)
    pb.end_frame_all(gs)
    print(it, [s.stats()['live'] for s in gs], flush=True)
