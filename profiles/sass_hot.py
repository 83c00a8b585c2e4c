"""Hottest SASS lines of an `ncu --page source --csv --print-source sass`
export (gzip ok): python profiles/sass_hot.py file.csv[.gz] [top]"""
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
op = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(op(path, "rt")))
h = rows[1]
si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for i, r in enumerate(rows[2:]):
    try:
        data.append((float(r[si] or 0), float(r[ie] or 0), i, r[1].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
print(f"{len(data)} SASS lines, {tot:.0f} stall samples, {toti:.3g} warp instructions executed")
for d in sorted(data, reverse=True)[:top]:
    print(f"{100 * d[0] / tot:5.1f}%  {d[1]:10.0f}  #{d[2]:5d}  {d[3][:90]}")
ops = {}
for s, n, _, src in data:
    o = src.split()[0] if src else "?"
    if o.startswith("@"):
        o = src.split()[1]
    o = o.split(".")[0]
    ops[o] = ops.get(o, 0) + n
print("dynamic mix (warp instructions):",
      ", ".join(f"{k} {100 * v / toti:.1f}%" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:14]))
