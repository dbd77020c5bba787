"""Attribute ncu per-SASS-instruction metrics (``--page source --csv
--print-source sass``) to the kernel's OUTERMOST source lines, using the
inlined-at chains of ``nvdisasm -gi`` on the same cubin.

    python tools/sass_attr.py ncu_sass.csv disasm_gi.txt kernel_mangled_name [top_file]
"""
import csv
import re
import sys
from collections import defaultdict

csv_path, dis_path, kernel = sys.argv[1], sys.argv[2], sys.argv[3]
top = sys.argv[4] if len(sys.argv) > 4 else "conv2d_kernels.cuh"
lines = []
inside, cur = False, None
for ln in open(dis_path):
    if ln.startswith("//----") and ".text." in ln:
        inside = ln.strip().endswith(kernel + " --------------------------") or (".text." + kernel + " ") in ln
        continue
    if not inside:
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', ln)
    if m:
        if "inlined at" not in m.group(3):
            cur = f'{m.group(1).split("/")[-1]}:{m.group(2)}'
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
        lines.append(cur)
rows = list(csv.reader(open(csv_path)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
col = {h: i for i, h in enumerate(hdr)}
if len(data) != len(lines):
    print(f"warning: {len(data)} ncu rows vs {len(lines)} disassembled instructions")
inst = defaultdict(float)
samp = defaultdict(float)
for r, key in zip(data, lines):
    inst[key] += float(r[col["Instructions Executed"]] or 0)
    samp[key] += float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
ti, ts = sum(inst.values()), sum(samp.values())
print(f"instructions executed {ti:.0f}, stall samples {ts:.0f}")
for k in sorted(inst, key=lambda k: -samp[k])[:40]:
    print(f"{k:32s} inst {100 * inst[k] / ti:5.1f}%  samples {100 * samp[k] / ts:5.1f}%")
