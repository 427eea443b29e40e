"""Aggregate an ncu source page (--print-source=cuda,sass --csv) per CUDA source line:
instructions executed and warp-stall samples. Usage: python tools/ncu_lines.py page.csv [top] [inst|stall]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
cur = None
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        continue
    if r[0].isdigit() and r[2] == "-":      # a CUDA source line with its aggregated metrics
        cur = (fname, int(r[0]))
        d = dict(zip(hdr, r))
        agg[cur][2] = r[1].strip()[:70]
        try:
            agg[cur][0] += float(d.get("Instructions Executed", 0) or 0)
            agg[cur][1] += float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        except ValueError:
            pass
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
key = 0 if (len(sys.argv) > 3 and sys.argv[3] == "inst") else 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    print(f"{k[0]}:{k[1]:<5d} inst {100*v[0]/tot_i:5.1f}%  stall {100*v[1]/tot_s:5.1f}%  {v[2]}")
