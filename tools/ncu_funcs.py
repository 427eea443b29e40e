"""Aggregate an ncu cuda,sass source page per device function of eval.cuh (by line ranges)."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
src = open(sys.argv[2]).read().split("\n")
hdr = None
fname = ""
agg = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 6 and r[0].isdigit() and r[2] == "-":
        d = dict(zip(hdr, r))
        agg[(fname, int(r[0]))] = (float(d["Instructions Executed"] or 0),
                                   float(d["Warp Stall Sampling (All Samples)"] or 0))
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r"(__device__|__global__)[^(]*?(\w+)\(", l)
    if m:
        starts.append((i, m.group(2)))


def fn(line):
    name = "?"
    for st, nm in starts:
        if st <= line:
            name = nm
    return name


tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
by = {}
base = sys.argv[2].split("/")[-1]
for (f, l), (i, s) in agg.items():
    k = fn(l) if f == base else f
    a = by.setdefault(k, [0, 0])
    a[0] += i
    a[1] += s
print(f"total instructions {tot:.3e}")
for k, v in sorted(by.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:32s} inst {100 * v[0] / tot:5.1f}%  stall {100 * v[1] / tots:5.1f}%")
