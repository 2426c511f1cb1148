import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2005_07547_b200 as pb
base = 12 ** 0.5 / 256
fs = pb.FieldStore(pb.FieldStoreConfig(capacity_log2=10, base_cell_size=base))
buf, n = pb.synth_generate(1920, 1080, 4)
f = buf[:34 * n].view(34, n)
flags = buf.view(torch.uint8)[34 * n * 8:34 * n * 8 + 4 * n].view(torch.int32)
lv = fs.select_level_batch(f[15])
for name, d, m in (("Lo", f[3:6], torch.ones(n, dtype=torch.bool, device="cuda")), ("FLi-cont", f[6:9], (flags & 1) != 0), ("FLi-nee", f[12:15], (flags & 4) != 0)):
    k = fs.key_for_batch(f[0:3], d, lv)[m]
    u, c = torch.unique(k[:, :6], dim=0, return_counts=True)
    print(name, "keys", u.shape[0], "max records per key", int(c.max()), "top5", c.sort(descending=True).values[:5].tolist())
