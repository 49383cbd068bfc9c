"""Where the C2 single-hypothesis latency goes (host wall times, p50 over reps)."""
import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2412_00802_b200 as hedl
from synth import abox, hyps
from synth.format import flatten
kb = abox.c2_kb()
nodes, kids, roots = flatten(hyps.c2_hypotheses(kb))
k = hedl.hedl_kb_load(kb, 0)
prog = hedl.hedl_compile(k, nodes, kids, roots)
L = hedl.lib()
def p50(f, n=2000):
    for _ in range(50): f()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return round(float(np.median(ts)) * 1e6, 2)
import ctypes as C
out = np.zeros(4, dtype=np.uint64)
st = torch.cuda.current_stream().cuda_stream
print('ctypes hedl_version', p50(lambda: L.hedl_version()))
print('torch.cuda.synchronize', p50(lambda: torch.cuda.synchronize()))
print('eval_one via binding', p50(lambda: hedl.hedl_eval_one(k, prog, 3)))
print('eval_one raw ctypes', p50(lambda: L.hedl_eval_one(k._h, prog._h, 3, None, out.ctypes.data, C.c_void_p(st))))
hedl.prof_reset(); hedl.prof_enable(True)
for _ in range(200): L.hedl_eval_one(k._h, prog._h, 3, None, out.ctypes.data, C.c_void_p(st))
hedl.prof_enable(False)
pr = hedl.prof_read()
print('kernel event time per call us', [(e['name'], round(e['total_ms'] * 1e3 / e['launches'], 2)) for e in pr])
x = torch.zeros(1, device='cuda')
print('torch tiny kernel + sync', p50(lambda: (x.add_(1), torch.cuda.synchronize())))
