"""SASS opcode mix of an ncu source page (--print-source=cuda,sass --csv), optionally restricted to
CUDA source lines [a, b] of one file. Usage: python tools/ncu_ops.py page.csv [file a b] [div]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
sel = (sys.argv[2], int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else None
div = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
fname, cur, ops = "", None, defaultdict(float)
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]))
        continue
    if r[2] in ("", "...") or cur is None:
        continue
    if sel and not (cur[0] == sel[0] and sel[1] <= cur[1] <= sel[2]):
        continue
    try:
        n = float(r[7])
    except ValueError:
        continue
    t = r[3].split()
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += n
tot = sum(ops.values())
print(f"total {tot / div:.0f}")
for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:40]:
    print(f"  {k:10s} {v / div:8.1f}")
