"""Diagnose the test_gpu_split oracle OUT_OF_RANGE on the GPU box (one-off)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
from oracle import setsem
from synth import abox, hyps
from synth.format import flatten
kb = abox.powerlaw_kb(120_000, 50, 2, 8.0, 3000, 0.7, 1.0, 0.01, seed=21)
print("shape", abox.kb_shape(kb), "cpus", os.cpu_count())
rng = np.random.default_rng(4)
t = [hyps.random_tree(rng, abox.kb_shape(kb), depth=5) for _ in range(40)] + hyps.c3_hypotheses()
nodes, kids, roots = flatten(t)
for th in (1, os.cpu_count()):
    try:
        setsem.evaluate(kb, nodes, kids, roots, threads=th); print("ok threads", th)
    except Exception as e:
        print("threads", th, e, "tree", t[47] if len(t) > 47 else None)
import paper_2412_00802_b200 as hedl
from paper_2412_00802_b200 import dist as hdist
plan = hdist.SplitPlan(nodes, kids, roots, kb["concept_bits"].shape[0])
try:
    setsem.evaluate(kb, nodes, kids, roots, threads=1); print("ok after SplitPlan")
except Exception as e:
    print("after SplitPlan", e)
