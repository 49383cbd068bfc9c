"""Per-class DRAM traffic of one bench step, from an ncu launch list of EVERY launch of the step.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --clock-control none --cache-control none --csv --log-file gpurun_out/traffic_c4.csv \\
        python bench.py --workload c4 --steps 1 --warmup 0 --no-prof-pass --no-e2e \\
        --no-cpu-baseline --no-latency --no-c5
    python tools/ncu_traffic.py gpurun_out/traffic_c4.csv c4 1 [profiles/ncu_traffic.json]

The bench command runs exactly `steps` steps (argv[3]) of the workload; every launch of the
library's kernels is attributed to the bench's profiling class (the names hedl_prof_read
reports), and the file records per class the launches per step, the measured DRAM bytes
(read + write) per launch and per step, and the whole step's DRAM bytes -- the numbers
bench.py reports as `roofline.traffic` and `roofline.step_dram_frac`.  `--cache-control none`
keeps the caches warm across launches as in the timed run (ncu's default flushes them before
every launch, which would charge L2-resident re-reads to DRAM); the three metrics need one pass.
"""
from __future__ import annotations

import csv
import json
import os
import re
import sys
from collections import defaultdict

# ncu kernel name (template arguments printed as 0/1) -> bench.py / hedl_prof_read class
CLASS_OF = [
    (r"^k_bool(_warp)?<1>", "bool"), (r"^k_bool(_warp)?<0>", "bool_l2"),
    (r"^k_slice_pack", "slice_pack"), (r"^k_slice_tile", "slice"), (r"^k_slice_heavy", "slice_heavy"),
    (r"^k_slice_ex", "slice_ex"), (r"^k_restrict_tile", "restrict"), (r"^k_restrict_heavy", "restrict_heavy"),
    (r"^k_drange", "drange"), (r"^k_cover_init", "cover_init"), (r"^k_gather_", "gather"),
    (r"^k_string", "string"), (r"^k_interp", "interp"),
]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
        "ns": 1e-3, "us": 1.0, "ms": 1e3}


def short_name(k: str) -> str:
    k = k.replace("void ", "")
    k = re.sub(r"\(anonymous namespace\)::", "", k)
    k = k.split("(")[0]
    return k.split("::")[-1]


def classify(name: str):
    for pat, cls in CLASS_OF:
        if re.match(pat, name):
            return cls
    return None


def parse(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Value" in r:
            hdr, body = r, rows[i + 1:]
            break
    else:
        raise SystemExit(f"{path}: no ncu CSV header")
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    ii = hdr.index("ID") if "ID" in hdr else None
    launches = defaultdict(dict)
    for n, r in enumerate(body):
        if len(r) <= vi:
            continue
        key = r[ii] if ii is not None else n
        v = float(r[vi].replace(",", ""))
        u = r[ui] if ui is not None else ""
        launches[key]["name"] = short_name(r[ki])
        launches[key][r[mi]] = v * UNIT.get(u, 1.0)
    return list(launches.values())


def main():
    path, workload, steps = sys.argv[1], sys.argv[2], int(sys.argv[3])
    out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                             "ncu_traffic.json")
    acc = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "time_us": 0.0})
    other = 0.0
    for L in parse(path):
        cls = classify(L["name"])
        b = L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0)
        if cls is None:
            other += b
            continue
        a = acc[cls]
        a["launches"] += 1
        a["dram_bytes"] += b
        a["time_us"] += L.get("gpu__time_duration.sum", 0.0)
    classes = {c: {"launches_per_step": a["launches"] / steps,
                   "dram_bytes_per_launch": a["dram_bytes"] / max(1, a["launches"]),
                   "dram_bytes_per_step": a["dram_bytes"] / steps,
                   "ncu_time_us_per_step": a["time_us"] / steps}
               for c, a in sorted(acc.items(), key=lambda kv: -kv[1]["dram_bytes"])}
    db = json.load(open(out)) if os.path.exists(out) else {}
    if "classes" not in db.get(workload, {}) and workload in db:
        del db[workload]
    db = {k: v for k, v in db.items() if isinstance(v, dict) and "classes" in v}
    db[workload] = {
        "source": f"{os.path.basename(path)}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                  "gpu__time_duration.sum --clock-control none --cache-control none, every launch of "
                  f"{steps} bench step(s)",
        "steps": steps, "classes": classes,
        "dram_bytes_per_step": sum(c["dram_bytes_per_step"] for c in classes.values()),
        "other_kernels_dram_bytes_per_step": other / steps,
    }
    json.dump(db, open(out, "w"), indent=1)
    print(json.dumps(db[workload], indent=1))


if __name__ == "__main__":
    main()
