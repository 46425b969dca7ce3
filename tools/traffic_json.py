"""profiles/traffic.json from `ncu --set full ... --page raw --csv` exports:
per launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the
roofline kernels, read by bench.py's `roofline.traffic`.

    python tools/traffic_json.py <tag> c4_large_sharded_bf16_xchg=<c4_raw.csv> c2_mid_bf16=<c2_raw.csv> ...

Roles: "gather" = the kernel that gathers the value rows (cartesian_route_kernel
on the sharded path, cartesian_gather_kernel / gather_kernel otherwise);
"dv_reduce" = grp_reduce_short_kernel<0, ...> (the dV reducer).
"""
import csv
import json
import os
import sys

ROLES = {"gather": ("cartesian_route_kernel", "cartesian_gather_kernel", "cartesian_gather_lookup_kernel", "gather_wide_kernel", "gather_kernel"),
         "dv_reduce": ("grp_reduce_short_kernel<0",)}


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)


def per_kernel(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        rd = float(r[ix["dram__bytes_read.sum"]].replace(",", "")) * unit_scale(units[ix["dram__bytes_read.sum"]])
        wr = float(r[ix["dram__bytes_write.sum"]].replace(",", "")) * unit_scale(units[ix["dram__bytes_write.sum"]])
        out.append((r[ix["Kernel Name"]], rd, wr))
    return out


def main():
    tag = sys.argv[1]
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    tj = json.load(open(path)) if os.path.exists(path) else {}
    for arg in sys.argv[2:]:
        key, raw = arg.split("=", 1)
        ks = per_kernel(raw)
        ent = {}
        notes = []
        for role, names in ROLES.items():
            for name, rd, wr in ks:
                if any(n in name for n in names):
                    ent[role] = int(rd + wr)
                    notes.append(f"{role}: {name.split('(')[0][-60:]} {rd / 1e6:.2f} + {wr / 1e6:.2f} MB")
                    break
        ent["_source"] = f"ncu --set full ({tag}): dram__bytes_read.sum + dram__bytes_write.sum per launch; " + "; ".join(notes)
        tj[key] = ent
    tj["_source"] = "ncu --set full per-launch DRAM bytes of the roofline kernels (tools/traffic_json.py)"
    json.dump(tj, open(path, "w"), indent=1)
    print(json.dumps(tj, indent=1))


if __name__ == "__main__":
    main()
