"""Summarise tools/ab.sh outputs: ms/step and per-launch kernel times per variant and repetition."""
import glob
import json
import os

for f in sorted(glob.glob("gpurun_out/ab_*_[12].json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(os.path.basename(f), "no result", e)
        continue
    k = {x["name"]: x for x in d["kernels"]}
    per = {n: round(1000 * x["total_ms"] / x["launches"], 1) for n, x in k.items() if x["launches"]}
    print(os.path.basename(f)[3:-5], round(d["ms_per_step"], 2), "ms/step", per)
for f in sorted(glob.glob("gpurun_out/ab_*_pytest.log")):
    print(os.path.basename(f), open(f).read().strip().splitlines()[-2:])
