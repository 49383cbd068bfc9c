"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times, on outputs the
oracle can compute one by one (SURVEY 8(d) "Parity protocol per config").

* C4: 10^6 individuals x 10^6 refinement hypotheses, evaluated exactly like bench.py's `value`
  (device counts, default flags); counts of a seeded sample of roots and bitsets of a smaller
  sample compared with the oracle; counts-only and bitset runs agree with each other.
* C3: 10^7 individuals, 1.6*10^8 assertions: the 8 fixed hypotheses, bitsets and counts.
* C5: 1.25*10^7 individuals, 10^8-edge role: a 20k cardinality/datatype-heavy batch, sampled.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import setsem
from synth import abox, hyps
from synth.format import flatten

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _hedl():
    import paper_2412_00802_b200 as hedl
    hedl.lib()
    return hedl


def test_c4_full_batch_sampled():
    import torch
    import bench
    hedl = _hedl()

    class A:
        n_individuals, n_hyps, seed, cache = 1_000_000, 1_000_000, 4, "/tmp/hedl_cache"
    kb_np, nodes, kids, roots = bench.c4_inputs(A, 1)
    kb = hedl.hedl_kb_load(kb_np, 0)
    prog = hedl.hedl_compile(kb, nodes, kids, roots)
    n = len(roots)
    counts = torch.empty((n, 4), dtype=torch.int64, device="cuda:0")
    hedl.hedl_eval_batch(kb, prog, 0, n, counts_device=True, out_counts=counts)      # bench's value path
    torch.cuda.synchronize()
    c_dev = counts.cpu().numpy().view(np.uint64)
    _, c_host = hedl.hedl_eval_batch(kb, prog, 0, n)                                  # bench's e2e path
    assert np.array_equal(c_dev, c_host)
    rng = np.random.default_rng(2024)
    sample = np.sort(rng.choice(n, 400, replace=False))
    okb = setsem.OracleKB(kb_np)
    _, oc = okb.evaluate(nodes, kids, roots[sample], want_bits=False, threads=os.cpu_count())
    assert np.array_equal(c_dev[sample], oc)
    # bitsets of a smaller sample through a separate program (bitsets requested -> full rows)
    bs = sample[:64]
    p2 = hedl.hedl_compile(kb, nodes, kids, roots[bs])
    gb, gc = hedl.hedl_eval_batch(kb, p2, 0, len(bs), want_bits=True)
    ob, oc2 = okb.evaluate(nodes, kids, roots[bs], want_bits=True, threads=os.cpu_count())
    assert np.array_equal(gb.cpu().numpy().view(np.uint32), ob) and np.array_equal(gc, oc2)


def test_c3_fixed_hypotheses():
    hedl = _hedl()
    kb_np = abox.c3_kb()
    trees = hyps.c3_hypotheses()
    nodes, kids, roots = flatten(trees)
    kb = hedl.hedl_kb_load(kb_np, 0)
    prog = hedl.hedl_compile(kb, nodes, kids, roots)
    gb, gc = hedl.hedl_eval_batch(kb, prog, 0, len(roots), want_bits=True)
    ob, oc = setsem.evaluate(kb_np, nodes, kids, roots, threads=os.cpu_count())
    assert np.array_equal(gc, oc)
    assert np.array_equal(gb.cpu().numpy().view(np.uint32), ob)
    for i in range(len(roots)):                    # the latency path (per-node kernels at this N)
        b1, c1 = hedl.hedl_eval_one(kb, prog, i, want_bits=True)
        assert c1 == tuple(int(v) for v in oc[i])
        assert np.array_equal(b1.cpu().numpy().view(np.uint32), ob[i])


def test_c5_card_datatype_sampled():
    hedl = _hedl()
    kb_np = abox.c5_kb()
    nodes, kids, roots = hyps.batch_arrays("c5", kb_np, 20_000, 5)
    kb = hedl.hedl_kb_load(kb_np, 0)
    prog = hedl.hedl_compile(kb, nodes, kids, roots)
    _, gc = hedl.hedl_eval_batch(kb, prog, 0, len(roots))
    rng = np.random.default_rng(5)
    sample = np.sort(rng.choice(len(roots), 120, replace=False))
    _, oc = setsem.evaluate(kb_np, nodes, kids, roots[sample], want_bits=False, threads=os.cpu_count())
    assert np.array_equal(gc[sample], oc)
