"""Summarise tools/ab2.sh outputs: ms/step and per-class ms/step per variant and repetition."""
import glob, json, os, sys
tag = sys.argv[1] if len(sys.argv) > 1 else "ab2"
for f in sorted(glob.glob(f"gpurun_out/{tag}_*.json")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    except Exception as e:
        print(os.path.basename(f), "no result"); continue
    print(os.path.basename(f)[len(tag) + 1:-5], round(d["ms_per_step"], 3), "ms/step",
          {k["name"]: round(k["ms_per_step"], 3) for k in d.get("kernels", [])[:7]})
for f in sorted(glob.glob(f"gpurun_out/{tag}*pytest.log")) + sorted(glob.glob(f"gpurun_out/{tag}chk_*.log")):
    print(os.path.basename(f), open(f).read().strip().splitlines()[-2:])
