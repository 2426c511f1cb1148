"""Per-function SASS instruction counts of a cubin/.so (cuobjdump -sass), for code-size checks."""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
fn, counts = None, {}
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        fn = m.group(1)
        counts[fn] = 0
    elif fn and re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
        counts[fn] += 1
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for f, c in sorted(counts.items(), key=lambda kv: -kv[1]):
    if pat in f:
        print(c, f)
