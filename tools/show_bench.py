"""Print the key numbers of a bench.py JSON line (file argument: the last JSON line is used)."""
import json
import sys

line = [l for l in open(sys.argv[1]) if l.startswith("{")][-1]
d = json.loads(line)
print("value %.4g hyps/s  ms/step %.3f  profiled %.3f" % (d["value"], d["ms_per_step"], d.get("profiled_ms_per_step") or 0))
if d.get("e2e"):
    e = d["e2e"]
    sm = sorted(e.get("step_ms", []))
    print("e2e %.4g hyps/s  ms %.2f  median step %.2f" % (e["value"], e["ms_per_step"], sm[len(sm) // 2] if sm else 0))
for k in d.get("kernels", []):
    print("  %-14s %7.3f ms  %5.1f launches  frac %.3f" % (k["name"], k["ms_per_step"], k["launches_per_step"], k["frac_of_hbm"]))
for w in ("c5",):
    if isinstance(d.get(w), dict) and "value" in d[w]:
        print("%s: %.4g hyps/s  ms/step %.2f" % (w, d[w]["value"], d[w]["ms_per_step"]))
