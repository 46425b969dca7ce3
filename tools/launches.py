"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"][:90]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    if unit in ("msecond", "ms"): v *= 1e3
    elif unit in ("nsecond", "ns"): v /= 1e3
    elif unit in ("second", "s"): v *= 1e6
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1; a[1] += v
tot = sum(v for _, v in agg.values())
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v:10.1f} us  {c:5d}x  {v/c:9.2f} us/launch  {100*v/tot:5.1f}%  {n}")
