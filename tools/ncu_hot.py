"""Hottest SASS instructions of one kernel in an ncu report (stall samples),
with the running instruction index for locating them:

    python tools/ncu_hot.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
ai, si, ni = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
body = []  # the first matching kernel's instructions (up to the next kernel's header)
for r in rows[rows.index(hdr) + 1:]:
    if r and r[0] in ("Address", "Kernel Name"):
        break
    if len(r) == len(hdr):
        body.append(r)
tot = sum(int(r[ni]) for r in body)
print(f"{len(body)} instructions, {tot} samples")
ranked = sorted(enumerate(body), key=lambda x: -int(x[1][ni]))[:top]
for i, r in ranked:
    print(f"{i:5d} {int(r[ni]):7d} {100.0 * int(r[ni]) / max(tot, 1):5.1f}%  {r[si].strip()[:90]}")
