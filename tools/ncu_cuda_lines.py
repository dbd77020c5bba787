"""Per-CUDA-line (innermost) executed instructions and stall samples from
`ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur, hdr, agg = None, None, {}
for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        col = {h: i for i, h in enumerate(r)}
        continue
    if hdr and cur and len(r) == len(hdr) and r[2] == "-":
        try:
            ie = float(r[col["Instructions Executed"]] or 0)
            sm = float(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        if ie or sm:
            k = (cur, int(r[0]))
            a = agg.get(k, (0.0, 0.0, r[1].strip()[:90]))
            agg[k] = (a[0] + ie, a[1] + sm, a[2])
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print(f"total instructions {ti:.0f}, samples {ts:.0f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k[0]}:{k[1]:<5d} inst {100 * v[0] / ti:5.1f}% samp {100 * v[1] / ts:5.1f}%  {v[2]}")
