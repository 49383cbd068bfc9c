import sys, os, numpy as np
sys.path.insert(0,'.')
import paper_2412_00802_b200 as hedl
from synth import abox
from synth.format import flatten
from oracle import setsem
kb = abox.powerlaw_kb(400_000, 12, 2, 8.0, 4000, 0.7, 1.0, 0.01, seed=31)
N=kb['N']
A=lambda i:("ATOM",i)
trees = []
for r in range(2):
    for inv in (False, True):
        for c in (A(0), A(5), A(11), ("NOT", A(3)), ("TOP",), ("BOTTOM",), ("AND", [A(1), A(2)])):
            trees += [("EXISTS", r, inv, c), ("FORALL", r, inv, c), ("MIN", 2, r, inv, c), ("MAX", 1, r, inv, c),
                      ("EXACT", 3, r, inv, c), ("MIN", 0, r, inv, c)]
nodes,kids,roots=flatten(trees)
k=hedl.hedl_kb_load(kb,0)
prog=hedl.hedl_compile(k,nodes,kids,roots)
ob,oc=setsem.evaluate(kb,nodes,kids,roots,threads=8)
bad=[]
for i in range(len(roots)):
    b,c=hedl.hedl_eval_one(k,prog,i,want_bits=True)
    g=np.unpackbits(b.cpu().numpy().view(np.uint8),bitorder='little')[:N]
    o=np.unpackbits(ob[i].view(np.uint8),bitorder='little')[:N]
    d=np.nonzero(g!=o)[0]
    if len(d): bad.append(i); print(i, trees[i], 'gpu ones',g.sum(),'oracle',o.sum(),'diff',len(d), d[:8], 'gpu', g[d[:8]], flush=True)
print('bad', bad)
# rerun the bad ones
for i in bad[:3]:
    b,c=hedl.hedl_eval_one(k,prog,i,want_bits=True)
    g=np.unpackbits(b.cpu().numpy().view(np.uint8),bitorder='little')[:N]
    o=np.unpackbits(ob[i].view(np.uint8),bitorder='little')[:N]
    print('rerun', i, (g!=o).sum())
