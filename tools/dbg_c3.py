"""Per-kernel-class times of the C3 latency path (one hedl_eval_one per hypothesis)."""
import sys, time, json, numpy as np
sys.path.insert(0, '.')
import bench, paper_2412_00802_b200 as hedl
from synth import abox, hyps
from synth.format import flatten
kb_np = bench._cached('/tmp/hedl_cache', 'c3kb_3', lambda: {k: np.asarray(v) for k, v in abox.c3_kb().items()})
kb_np['N'] = int(kb_np['N'])
nodes, kids, roots = flatten(hyps.c3_hypotheses())
k = hedl.hedl_kb_load(kb_np, 0)
prog = hedl.hedl_compile(k, nodes, kids, roots)
for i in range(len(roots)):
    for _ in range(3): hedl.hedl_eval_one(k, prog, i)
    hedl.prof_reset(); hedl.prof_enable(True)
    t0 = time.perf_counter(); hedl.hedl_eval_one(k, prog, i); t = time.perf_counter() - t0
    hedl.prof_enable(False)
    pr = hedl.prof_read()
    print(i, round(t * 1e6, 1), [(e['name'], e['launches'], round(e['total_ms'] * 1e3, 1)) for e in pr], flush=True)
