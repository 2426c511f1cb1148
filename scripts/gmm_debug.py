import sys, os
sys.path[:0]=[os.getcwd()+'/tests', os.getcwd()+'/oracle', os.getcwd()]
import numpy as np, torch, pyoracle as po, model_cases as mc, paper_2005_07547_b200 as pb
comps, alpha, skew = 3, 0.95, 1.0
SPLIT = int(os.environ.get('SPLIT', '1'))
rng = np.random.default_rng(comps * 13 + int(alpha * 100))
g = pb.ModelStore(16, 64.0, 4, capacity_log2=10, kind=pb.MODEL_GMM, gmm_components=comps, gmm_alpha_em=alpha)
r = po.RefModelStore(16, 64.0, 4, kind=2, comps=comps, alpha_em=alpha)
C=comps
names=[f"W{c}" for c in range(C)]+[f"M{c}{a}" for c in range(C) for a in "xy"]+[f"V{c}{a}" for c in range(C) for a in ("xx","xy","yy")]+[f"U{c}_{q}" for c in range(C) for q in range(8)]+[f"K{c}_{q}" for c in range(C) for q in range(7)]
for frame in range(5):
    k, u, v, c, keys = mc.model_records(rng, 4000, 120, skew=skew)
    perm = rng.permutation(len(k)); half = len(k)//2
    if SPLIT:
        g.apply(k[:half], u[:half], v[:half], c[:half]); g.apply(k[half:], u[half:], v[half:], c[half:])
        r.apply(k[:half], u[:half], v[:half], c[:half]); r.apply(k[half:], u[half:], v[half:], c[half:])
    else:
        g.apply(k, u, v, c); r.apply(k, u, v, c)
    if os.environ.get('ORACLE'):
        pass
    g.end_frame(); r.end_frame()
    eg, sg, _ = g.dump(); er, sr, _ = r.dump()
    rel = np.abs(sg[:, :21*C]-sr[:, :21*C]) / (np.abs(sr[:, :21*C]) + 1e-12)
    bad = np.argwhere(rel > 1e-9)
    print("frame", frame, "max rel", rel.max(), "bad", len(bad))
    for (i, j) in bad[:12]:
        print("  entry", i, names[j], sg[i, j], sr[i, j], "records", er['records'][i], "i", sr[i,21*C])
