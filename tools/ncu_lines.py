"""Per-source-line stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur = None
agg = {}
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and cur and len(r) > 6 and r[2] == "-":     # source-line aggregate rows
        try:
            s = float(r[4] or 0)
        except ValueError:
            continue
        key = (cur, r[0])
        agg[key] = (agg.get(key, (0, r[1]))[0] + s, r[1])
tot = sum(v[0] for v in agg.values())
print(f"total {tot:.0f}")
for (f, l), (s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100 * s / tot:5.1f}% {f}:{l:5s} {src.strip()[:100]}")
