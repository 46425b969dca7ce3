"""Per-kernel SASS instruction census of the built library (evidence that the
hot kernels are tcgen05 / TMA / TMEM code): counts of UTCHMMA / UTCQMMA (tcgen05
MMA), UTMALDG / UBLKCP (TMA / bulk copies), LDTM / STTM (TMEM loads / stores),
SYNCS (mbarrier), and the total per kernel.

    python tools/sass_summary.py [libmsn_pkm.so] > profiles/r02_sass_summary.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2602_07526_b200", "libmsn_pkm.so")
out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "UTCMMA", "UTMALDG", "UBLKCP", "LDTM", "STTM", "SYNCS", "REDG", "LDG", "STG"]
fn, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        fn = m.group(1)
        counts[fn] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if fn and m:
        op = m.group(1).split(".")[0]
        counts[fn]["total"] += 1
        for k in KEYS:
            if op == k:
                counts[fn][k] += 1


def short(name):
    try:
        d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        d = name
    d = re.sub(r"msn::\(anonymous namespace\)::", "", d)
    return d[:110]


print("%-110s %7s %8s %7s %6s %6s %6s" % ("kernel", "total", "UTC*MMA", "UTMALDG", "LDTM", "STTM", "SYNCS"))
tot = collections.Counter()
for f, c in counts.items():
    mma = c["UTCHMMA"] + c["UTCQMMA"] + c["UTCMMA"]
    tot.update(c)
    tot["mma"] += mma
    if mma or c["UTMALDG"] or c["LDTM"]:
        print("%-110s %7d %8d %7d %6d %6d %6d" % (short(f), c["total"], mma, c["UTMALDG"], c["LDTM"], c["STTM"],
                                                  c["SYNCS"]))
print("library totals: %d kernels, UTC*MMA %d, UTMALDG %d, LDTM %d, STTM %d" % (len(counts), tot["mma"], tot["UTMALDG"],
                                                                              tot["LDTM"], tot["STTM"]))
