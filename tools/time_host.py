"""Host-phase timing of compile + plan on the C4 batch (HEDL_TIMING=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HEDL_TIMING"] = "1"
import numpy as np, torch
import bench
import paper_2412_00802_b200 as hedl

class A: pass
a = A(); a.n_individuals = 1_000_000; a.n_hyps = 1_000_000; a.seed = 4; a.cache = "/tmp/hedl_cache"
kb_np, nodes, kids, roots = bench.c4_inputs(a, 1)
kb = hedl.hedl_kb_load(kb_np, 0)
for rep in range(2):
    t = time.perf_counter(); prog = hedl.hedl_compile(kb, nodes, kids, roots); t1 = time.perf_counter()
    _, c = hedl.hedl_eval_batch(kb, prog, 0, len(roots)); t2 = time.perf_counter()
    _, c = hedl.hedl_eval_batch(kb, prog, 0, len(roots)); t3 = time.perf_counter()
    print(f"compile {1e3*(t1-t):.1f} ms, first eval {1e3*(t2-t1):.1f} ms, cached eval {1e3*(t3-t2):.1f} ms", flush=True)
    prog.free()
