"""Summarise an ncu --page source --csv --print-source sass dump: stall
reasons overall and the hottest SASS instructions (with a little context)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
col = {h: i for i, h in enumerate(hdr)}
S = col["Warp Stall Sampling (All Samples)"]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in data:
    for h in stall_cols:
        try:
            tot[h] += float(r[col[h]] or 0)
        except ValueError:
            pass
allsamp = sum(float(r[S] or 0) for r in data)
print(f"total samples {allsamp:.0f}")
for h, v in tot.most_common(10):
    print(f"  {h:28s} {v:8.0f} {100 * v / max(allsamp, 1):5.1f}%")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 25
idx = sorted(range(len(data)), key=lambda i: -float(data[i][S] or 0))[:k]
for i in sorted(idx):
    r = data[i]
    top = sorted(((float(r[col[h]] or 0), h) for h in stall_cols), reverse=True)[:2]
    print(f"{r[0]:>8s} {float(r[S] or 0):7.0f}  {r[1][:70]:70s} {top[0][1]}={top[0][0]:.0f} {top[1][1]}={top[1][0]:.0f}")
