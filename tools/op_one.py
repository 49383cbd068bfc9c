"""One operator cell of tools/opbench.py, evaluated `reps` times through hedl_eval_one (for an
ncu launch list of the latency path): python tools/op_one.py exists unique 10000000 [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_00802_b200 as hedl  # noqa: E402
from synth import abox  # noqa: E402
from synth.format import flatten  # noqa: E402

op, regime, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
A = lambda i: ("ATOM", i)
tree = {"exists": ("EXISTS", 0, False, A(0)), "forall": ("FORALL", 0, False, A(0)),
        "min": ("MIN", 3, 0, False, A(0)), "max": ("MAX", 3, 0, False, A(0))}[op]
kb_np = abox.string_regime_kb(regime, n, seed=n)
k = hedl.hedl_kb_load(kb_np, 0)
nodes, kids, roots = flatten([tree])
prog = hedl.hedl_compile(k, nodes, kids, roots)
for _ in range(reps):
    b, c = hedl.hedl_eval_one(k, prog, 0, want_bits=True)
torch.cuda.synchronize()
print(op, regime, n, c)
