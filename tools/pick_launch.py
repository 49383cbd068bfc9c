"""From an ncu launch list (gpu__time_duration.sum CSV): the kernel with the largest total time
(or the kernel named by argv[2]) and, for it, the invocation index (among launches of that
kernel) with the largest grid.  Prints: <kernel-name-regex> <invocation-index>"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for i, r in enumerate(rows):
    if "Kernel Name" in r and "Metric Value" in r:
        hdr, body = r, rows[i + 1:]
        break
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
tot = defaultdict(float)
launches = defaultdict(list)
for r in body:
    if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
        continue
    name = r[ki].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
    v = float(r[vi].replace(",", ""))
    tot[name] += v
    g = [int(x) for x in r[gi].strip("()").split(",")]
    launches[name].append(g[0] * g[1] * g[2])
top = sys.argv[2] if len(sys.argv) > 2 else max(tot, key=tot.get)
sizes = launches[top]
idx = max(range(len(sizes)), key=lambda i: sizes[i])
print(top, idx)
