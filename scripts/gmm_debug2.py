"""GMM: compare split (two apply calls per frame) vs one call, GPU and reference."""
import os
import sys
sys.path[:0] = [os.getcwd() + '/tests', os.getcwd() + '/oracle', os.getcwd()]
import numpy as np  # noqa: E402
import model_cases as mc  # noqa: E402
import paper_2005_07547_b200 as pb  # noqa: E402
import pyoracle as po  # noqa: E402

comps, alpha, skew = 3, 0.95, 1.0
stores = {}
for name in ("g1", "g2", "r1", "r2", "o2"):
    if name[0] == "g":
        stores[name] = pb.ModelStore(16, 64.0, 4, capacity_log2=10, kind=pb.MODEL_GMM,
                                     gmm_components=comps, gmm_alpha_em=alpha)
    elif name[0] == "r":
        stores[name] = po.RefModelStore(16, 64.0, 4, kind=2, comps=comps, alpha_em=alpha)
    else:
        stores[name] = po.OracleModelStore(16, 64.0, 4, kind=2, comps=comps, alpha_em=alpha)
rng = np.random.default_rng(comps * 13 + int(alpha * 100))
for frame in range(4):
    k, u, v, c, keys = mc.model_records(rng, 4000, 120, skew=skew)
    if os.environ.get('CLEAN'):
        u = rng.random(len(k)); v = rng.random(len(k)); c = rng.exponential(1.0, len(k)) + 0.1
    rng.permutation(len(k))
    h = len(k) // 2
    for name, s in stores.items():
        if name.endswith("2"):
            s.apply(k[:h], u[:h], v[:h], c[:h])
            s.apply(k[h:], u[h:], v[h:], c[h:])
        else:
            s.apply(k, u, v, c)
        s.end_frame()
d = {n: s.dump()[1] for n, s in stores.items()}
for a, b in (("g2", "r2"), ("g1", "r1"), ("g2", "g1"), ("r2", "r1"), ("o2", "r2"), ("g2", "r1")):
    print(a, b, np.abs(d[a] - d[b]).max(), (np.abs(d[a] - d[b]) / (np.abs(d[b]) + 1e-300)).max())
