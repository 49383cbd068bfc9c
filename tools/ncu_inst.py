"""Per-source-line executed warp instructions of one kernel launch in an .ncu-rep:
python tools/ncu_inst.py REP [launch-skip] [top-n]"""
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
hdr = next(r for r in rows if len(r) > 4 and r[0] == "Line No")
ii = hdr.index("Instructions Executed")
agg, src, f = defaultdict(int), {}, "?"
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) > ii and r[0].isdigit():
        try:
            v = int(r[ii] or 0)
        except ValueError:
            continue
        agg[(f, int(r[0]))] += v
        src[(f, int(r[0]))] = r[1].strip()[:100]
tot = sum(agg.values())
print("total warp instructions", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v:10d} {100.0 * v / tot:5.1f}% {k[0]}:{k[1]} {src[k]}")
