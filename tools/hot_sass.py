"""Top stall-sampled SASS instructions from `ncu --page source --csv --print-source=sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[key] or 0) for d in data)
top = sorted(data, key=lambda d: -float(d[key] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for d in top:
    print(f"{100 * float(d[key] or 0) / tot:5.1f}%  {d['Address']:>6}  {d['Source'][:110]}")
