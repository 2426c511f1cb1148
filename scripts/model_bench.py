"""Model-store throughput on a config-2-shaped record stream: one CV-profile
record per continued vertex of the 1080p x 4 synthetic frame, keyed by the vertex's Lo key
(estimators.cpp:271-281), uv uniform on the square, exponential contributions.  Times
apply + endFrame per frame on the GPU (CUDA events) and the reference ModelStore compiled in
place (oracle/_ref, single thread as at the reference's frame barrier) on a bounded sample."""
import json
import os
import sys
import time

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_07547_b200 as pb  # noqa: E402

W, H, B = 1920, 1080, 4
base = 12 ** 0.5 / 256
keyer = pb.FieldStore(pb.FieldStoreConfig(capacity_log2=10, base_cell_size=base))


def frame_records(it, rng):
    buf, n = pb.synth_generate(W, H, B, iteration=it)
    f = buf[:34 * n].view(34, n)
    lv = keyer.select_level_batch(f[15])
    keys = keyer.key_for_batch(f[0:3], f[3:6], lv)
    cont = (buf.view(torch.uint8)[34 * n * 8:34 * n * 8 + 4 * n].view(torch.int32) & 1) != 0
    keys = keys[cont]
    m = keys.shape[0]
    g = torch.Generator(device="cuda").manual_seed(it)
    u = torch.rand(m, dtype=torch.float64, device="cuda", generator=g)
    v = torch.rand(m, dtype=torch.float64, device="cuda", generator=g)
    c = -torch.log(torch.rand(m, dtype=torch.float64, device="cuda", generator=g))
    return keys, u, v, c


res = int(os.environ.get("RES", "16"))
mode = pb.MODE_ATOMIC if os.environ.get("MODE", "ordered") == "atomic" else pb.MODE_ORDERED
kind = {"grid": pb.MODEL_GRID, "kdtree": pb.MODEL_KDTREE, "gmm": pb.MODEL_GMM}[os.environ.get("KIND", "grid")]
ms = pb.ModelStore(res, 64.0, 32, capacity_log2=int(os.environ.get("CAP", "22")), kind=kind)
rng = np.random.default_rng(0)
frames = [frame_records(i, rng) for i in range(6)]
for k, u, v, c in frames[:2]:  # warm-up (fills the table)
    ms.apply(k, u, v, c, mode=mode)
    ms.end_frame()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
t_apply = t_ef = 0.0
nrec = 0
for k, u, v, c in frames[2:]:
    ev[0].record()
    ms.apply(k, u, v, c, mode=mode)
    ev[1].record()
    ms.end_frame()
    ev[2].record()
    torch.cuda.synchronize()
    t_apply += ev[0].elapsed_time(ev[1])
    t_ef += ev[1].elapsed_time(ev[2])
    nrec += k.shape[0]
nf = len(frames) - 2
if os.environ.get("PROFILE"):
    pb.profile_enable(True)
    k, u, v, c = frames[2]
    ms.apply(k, u, v, c, mode=mode)
    ms.end_frame()
    prof = pb.profile_collect()
    pb.profile_enable(False)
    for name, (t, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        print(f"  {name[:40]:40s} {t:8.3f} ms x{cnt}")
st = ms.stats()
out = {"kind": ["grid", "kdtree", "gmm"][kind],
       "mode": "atomic" if mode == pb.MODE_ATOMIC else "ordered", "records_per_frame": nrec // nf, "entries": st["entries"], "warm": st["warm"],
       "grid_resolution": res, "apply_ms": t_apply / nf, "end_frame_ms": t_ef / nf,
       "gpu_records_per_s": nrec / ((t_apply + t_ef) / 1e3)}

import pyoracle as po  # noqa: E402  (checker / CPU baseline only)
if po.model_ref_available():
    k, u, v, c = frames[2]
    m = k.shape[0] // 16  # bounded sample: 1/16 of a frame
    kn = k[:m].cpu().numpy().view(po.KEY_DTYPE).reshape(m)
    r = po.RefModelStore(res, 64.0, 32, kind=kind)
    t0 = time.perf_counter()
    r.apply(kn, u[:m].cpu().numpy(), v[:m].cpu().numpy(), c[:m].cpu().numpy())
    r.end_frame()
    dt = time.perf_counter() - t0
    out["cpu_reference_records_per_s"] = m / dt
    out["cpu_sample"] = f"{m} records (1/16 of a frame), 1 thread, apply + endFrame"
print(json.dumps(out))
