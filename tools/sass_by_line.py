"""Attribute SASS instruction counts of one kernel to its outermost source
lines (nvdisasm -gi output): shows which call sites own the code size."""
import re
import sys
from collections import Counter

path, kernel = sys.argv[1], sys.argv[2]
top = sys.argv[3] if len(sys.argv) > 3 else "conv2d_kernels.cuh"
cnt = Counter()
inside = False
cur = None
pending = []
for line in open(path):
    if line.startswith("//----") and ".text." in line:
        inside = kernel in line
        continue
    if not inside:
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', line)
    if m:
        if "inlined at" not in m.group(3):
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
        cnt[cur] += 1
tot = sum(cnt.values())
print("total", tot)
for (f, l), n in sorted(cnt.items(), key=lambda kv: (str(kv[0][0]), kv[0][1])):
    if n >= 50:
        print(f"{f}:{l}  {n}")
