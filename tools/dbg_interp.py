import sys, os, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2412_00802_b200 as hedl
from tools.opbench import concepts_kb, measure
from synth import abox
for n in (30_000, 100_000, 1_000_000, 10_000_000):
    kb = abox.regime_kb("unique", n, seed=n)
    for name, tree in (("exists", ("EXISTS", 0, False, ("ATOM", 0))), ("and2", ("AND", [("ATOM", 0), ("NOT", ("ATOM", 1))]))):
        print(n, name, "default", measure(kb, tree, 20, False)[:2], flush=True)
