"""Aggregate an ncu source-page CSV (--print-source cuda,sass) by CUDA source line."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
byline = collections.defaultdict(lambda: [0.0, 0.0])
src = {}
fname = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        i_ex = hdr.index("Instructions Executed")
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr) or not r[0]:
        continue
    try:
        ln = int(r[0])
        ex = float(r[i_ex] or 0)
        s = float(r[i_s] or 0)
    except ValueError:
        continue
    key = (fname, ln)
    src[key] = r[1]
    byline[key][0] += ex
    byline[key][1] += s
tot_ex = sum(v[0] for v in byline.values()) or 1
tot_s = sum(v[1] for v in byline.values()) or 1
print("total warp instructions", tot_ex, "stall samples", tot_s)
for (fn, ln), (ex, s) in sorted(byline.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{fn[:14]:14s}:{ln:5d} inst {100 * ex / tot_ex:5.1f}% stall {100 * s / tot_s:5.1f}%  "
          f"{src[(fn, ln)].strip()[:80]}")
