"""Per-SASS-instruction view of `ncu -i rep --page source --csv -k regex:<kernel>`:
the top instructions by warp-stall samples and, with --regions N, the
executed-instruction / stall totals per block of N consecutive instructions.

    python tools/ncu_sass_top.py source.csv [top_n] [--regions N]
"""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    data = []
    for r in rows[hi + 1:]:
        if r and r[0] == "Address":
            break  # the next section repeats the header
        if len(r) == len(h):
            data.append(r)
    return h, data


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    h, data = load(args[0])
    top = int(args[1]) if len(args) > 1 else 30
    si = h.index("Warp Stall Sampling (All Samples)")
    ie = h.index("Instructions Executed")
    stot = sum(f(r[si]) for r in data) or 1.0
    itot = sum(f(r[ie]) for r in data) or 1.0
    print(f"instructions executed {itot:.0f}, stall samples {stot:.0f}, {len(data)} SASS lines")
    if "--regions" in sys.argv:
        n = int(sys.argv[sys.argv.index("--regions") + 1])
        for b in range(0, len(data), n):
            blk = data[b:b + n]
            s = sum(f(r[si]) for r in blk)
            e = sum(f(r[ie]) for r in blk)
            if s / stot > 0.01 or e / itot > 0.01:
                worst = max(blk, key=lambda r: f(r[si]))
                print(f"{b:5d} {100 * e / itot:5.1f}% inst {100 * s / stot:5.1f}% stall  {blk[0][1][:40]:40s} | {worst[1][:50]}")
        return
    for i, r in sorted(enumerate(data), key=lambda x: -f(x[1][si]))[:top]:
        print(f"{100 * f(r[si]) / stot:5.1f}%  #{i:<5d} {f(r[ie]):10.0f}  {r[1][:90]}")


if __name__ == "__main__":
    main()
