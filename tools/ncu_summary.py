"""Summarise an `ncu --page raw --csv` export: per kernel launch the duration,
DRAM bytes, DRAM/L2/SM throughput, tensor-pipe activity, occupancy, registers.

    python tools/ncu_summary.py raw.csv [more metric names...]
"""
import csv
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3),
        ("dram__bytes_read.sum", "MB_rd", 1e-6),
        ("dram__bytes_write.sum", "MB_wr", 1e-6),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%", 1),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
        ("lts__t_sectors_op_read.sum", "L2rd_sec", 1e-6),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%", 1),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tc%", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
        ("launch__registers_per_thread", "regs", 1),
        ("smsp__inst_executed.sum", "Minst", 1e-6)]


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units = rows[0], rows[1]
    extra = sys.argv[2:]
    cols = COLS + [(m, m.split("__")[-1][:14], 1) for m in extra]
    ix = {h: i for i, h in enumerate(hdr)}
    kn = ix.get("Kernel Name")
    print("%-48s" % "kernel" + "".join("%10s" % c[1] for c in cols))
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        line = "%-48s" % r[kn][:48]
        for m, _, sc in cols:
            i = ix.get(m)
            v = num(r[i]) if i is not None else None
            if v is not None and m == "gpu__time_duration.sum":
                u = units[i]
                v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
                sc = 1
            elif v is not None and units[i].endswith("byte"):
                # normalise to bytes, then the column scale (1e-6 -> MB)
                v = v * {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1.0)
            line += "%10.2f" % (v * sc) if v is not None else "%10s" % "-"
        print(line)


if __name__ == "__main__":
    main()
