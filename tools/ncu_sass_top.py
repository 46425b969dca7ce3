"""Top SASS instructions by warp-stall samples from
`ncu -i rep --page source --csv -k regex:<kernel>`.

    python tools/ncu_sass_top.py source.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
tot = sum(float(r[si] or 0) for r in data) or 1.0
for i, r in sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0))[:n]:
    print(f"{100 * float(r[si]) / tot:5.1f}%  #{i:<5d} {r[1][:100]}")
