"""SASS instruction counts per CUDA source line (and per line range) of one kernel, from
`nvdisasm -g` of the library's cubin: where the static code size of a kernel goes.

  python scripts/sass_lines.py paper_2005_07547_b200/lib/libpstf_b200.so k_vertex_pass_tiledILi1ELi4E [top]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

so, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True,
                         text=True).stdout.splitlines()
start = next(i for i, l in enumerate(txt) if re.match(r"\.text\.\S*" + pat + r"\S*:", l))
cnt, cur, total = collections.Counter(), None, 0
for l in txt[start + 1:]:
    if l.startswith("//----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
    elif re.match(r"\s*/\*[0-9a-f]{4,}\*/", l):
        cnt[cur] += 1
        total += 1
print("total", total)
byfile = collections.Counter()
for k, v in cnt.items():
    byfile[k[0] if k else None] += v
print(byfile.most_common())
for k, v in cnt.most_common(top):
    print(v, k)
