"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export by CUDA source line:
instructions executed and stall samples per line (the source rows carry the line totals)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
fname, hdr = None, None
recs = []
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
    if hdr is None or not r[0]:
        continue
    try:
        recs.append((fname, int(r[0]), r[1], float(r[i_ex] or 0), float(r[i_s] or 0)))
    except ValueError:
        pass
tex = sum(x[3] for x in recs) or 1
ts = sum(x[4] for x in recs) or 1
print("total warp instructions %.4g, stall samples %.4g" % (tex, ts))
byfile = collections.defaultdict(lambda: [0, 0])
for f, _, _, ex, s in recs:
    byfile[f][0] += ex
    byfile[f][1] += s
for f, (ex, s) in byfile.items():
    print(f"  {f}: inst {100*ex/tex:.1f}% stall {100*s/ts:.1f}%")
key = 4 if len(sys.argv) <= 3 or sys.argv[3] == "stall" else 3
for f, ln, src, ex, s in sorted(recs, key=lambda x: -x[key])[:top]:
    print(f"{f[:14]:14s}:{ln:5d} inst {100*ex/tex:5.1f}% stall {100*s/ts:5.1f}%  {src.strip()[:90]}")
