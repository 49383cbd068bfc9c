"""Per-source-line warp-stall samples of one kernel launch in an .ncu-rep (source/SASS
correlation view): python tools/ncu_hot.py REP [launch-skip] [top-n]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
lid = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip", lid,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, src, f = defaultdict(int), {}, "?"
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        continue
    if len(r) > 4 and r[0].isdigit():
        try:
            v = int(r[4] or 0)
        except ValueError:
            continue
        agg[(f, int(r[0]))] += v
        src[(f, int(r[0]))] = r[1].strip()[:100]
tot = sum(agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v:6d} {100.0 * v / tot:5.1f}% {k[0]}:{k[1]} {src[k]}")
