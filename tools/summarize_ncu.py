"""Summarise ncu outputs into profiles/ (launch list shares + `--set full` key metrics + traffic json)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Value" in r:
            hdr, body = r, rows[i + 1:]
            break
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = defaultdict(lambda: [0, 0.0])
    for r in body:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(a[1] for a in agg.values())
    return {k: {"launches": a[0], "total_us": round(a[1], 1), "share": round(a[1] / tot, 4)}
            for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])}


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ["launch__grid_size", "launch__grid_dim_y", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    ki = hdr.index("Kernel Name")
    res = []
    for r in rows[2:]:
        d = {"kernel": r[ki].split("(")[0].replace("void ", "").split("::")[-1]}
        for w, i in idx.items():
            d[w] = r[i] + " " + units[i]
        res.append(d)
    return res


def to_bytes(v):
    num, unit = v.split()[0], v.split()[1]
    return float(num.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


if __name__ == "__main__":
    launches, out_md, out_json = sys.argv[1:4]
    reps = sys.argv[4:]
    sh = launch_shares(launches)
    fm = []
    for rep in reps:
        fm += full_metrics(rep)
    with open(out_md, "w") as f:
        f.write("# ncu summary\n\n## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n\n")
        f.write("| kernel | launches | total us | share |\n|---|---|---|---|\n")
        for k, a in sh.items():
            f.write(f"| {k} | {a['launches']} | {a['total_us']} | {a['share']:.3f} |\n")
        f.write("\n## `ncu --set full` captures\n\n")
        keys = list(fm[0].keys()) if fm else []
        f.write("| " + " | ".join(keys) + " |\n|" + "---|" * len(keys) + "\n")
        for d in fm:
            f.write("| " + " | ".join(str(d.get(k, "")) for k in keys) + " |\n")
    name_map = {"k_slice_tile": "slice", "k_bool": "bool", "k_slice_pack": "slice_pack", "k_slice_ex": "slice_ex",
                "k_slice_heavy": "slice_heavy", "k_restrict": "restrict", "k_restrict_heavy": "restrict_heavy",
                "k_drange": "drange"}
    tj = defaultdict(list)
    for d in fm:
        try:
            tr = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
            gy = float(d.get("launch__grid_dim_y", "1 x").split()[0].replace(",", "") or 1)
            tj[name_map.get(d["kernel"].split("<")[0], d["kernel"])].append((tr, gy))
        except Exception as e:
            print("skip", d.get("kernel"), e)
    json.dump({k: {"dram_bytes_per_unit": sum(t for t, _ in v) / max(1.0, sum(g for _, g in v)),
                   "captures": len(v), "units_captured": sum(g for _, g in v)} for k, v in tj.items()},
              open(out_json, "w"), indent=1)
    print(open(out_md).read())
