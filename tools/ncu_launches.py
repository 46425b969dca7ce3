"""Summarise an `ncu --metrics ... --csv --log-file` launch list (one metric
per line): per launch the kernel, duration and DRAM bytes, in launch order,
and the step total.

    python tools/ncu_launches.py launches.csv
"""
import csv
import sys
from collections import OrderedDict

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
        "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def main():
    lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, ui, vi, ii = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    d = OrderedDict()
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        d.setdefault((r[ii], r[ki]), {})[r[mi]] = v
    tot = 0.0
    print("%-70s %10s %10s %10s" % ("kernel", "us", "MB_rd", "MB_wr"))
    for (_, k), m in d.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        tot += t
        print("%-70s %10.1f %10.1f %10.1f" % (k[:70], t, m.get("dram__bytes_read.sum", 0.0),
                                             m.get("dram__bytes_write.sum", 0.0)))
    print("%-70s %10.1f" % ("total (serialised, cold)", tot))


if __name__ == "__main__":
    main()
