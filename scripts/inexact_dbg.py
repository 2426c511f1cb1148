import sys
sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np
import pyoracle as po, inputs, gpu_util as gu
import paper_2005_07547_b200 as pb
from test_gpu_parity import _random_updates, _apply_gpu, _pcfg
for wkind in ["int", "frac"]:
  for tmax in [2.0, 64.0]:
    cfg = po.Config.make(capacity_log2=12, base_cell_size=0.5, probe_window=32, evict_age_frames=3, t_max=tmax)
    o = po.OracleStore(cfg); g = pb.FieldStore(_pcfg(cfg)); rng = np.random.default_rng(77)
    for f in range(4):
        u = _random_updates(o, rng, 18000, 3000)
        if wkind == "frac": u["w"] = rng.uniform(0.0, 3.0, size=len(u))
        o.queue_apply(u); _apply_gpu(g, u[rng.permutation(len(u))], pb.MODE_ORDERED)
        a, b = g.slots(), o.slots()
        pre = {k: int((gu.bits(a[k]).reshape(len(a), -1) != gu.bits(b[k]).reshape(len(b), -1)).any(1).sum()) for k in a.dtype.names}
        o.end_frame(); g.end_frame()
        a, b = g.slots(), o.slots()
        post = {k: int((gu.bits(a[k]).reshape(len(a), -1) != gu.bits(b[k]).reshape(len(b), -1)).any(1).sum()) for k in a.dtype.names}
        print(wkind, tmax, f, "pre", {k: v for k, v in pre.items() if v}, "post", {k: v for k, v in post.items() if v}, flush=True)
