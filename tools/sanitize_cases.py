"""Representative evaluations for compute-sanitizer runs (tools/sanitize.sh): every kernel family
of the library on small inputs, each result checked against the oracle so a sanitizer run is
also a parity run.

  C1 (every constructor): batch on the default / forced-pack / per-node paths, eval_one (the
  single-CTA interpreter), device compile + device plan;
  a random tiny KB with string roles (string kernels, EQUAL short-circuit);
  a 20k-individual power-law batch (lane packs: full, EX over U rows, heavy rows, fused
  fillers, U rows of restrictions and ranges; per-node kernels; device plan);
  scores + top-k on the device; hedl_kb_set_concept_rows.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2412_00802_b200 as hedl  # noqa: E402
from oracle import scores as oscores  # noqa: E402
from oracle import setsem  # noqa: E402
from synth import abox, hyps  # noqa: E402
from synth.format import flatten  # noqa: E402


def check(kb_np, nodes, kids, roots, eflags_list=(0,), tag="", device_compile=True, eval_one=()):
    import torch
    k = hedl.hedl_kb_load(kb_np, 0)
    ob, oc = setsem.evaluate(kb_np, nodes, kids, roots, threads=os.cpu_count())
    prog = hedl.hedl_compile(k, nodes, kids, roots)
    for ef in eflags_list:
        b, c = hedl.hedl_eval_batch(k, prog, 0, len(roots), want_bits=True, flags=ef)
        assert np.array_equal(b.cpu().numpy().view(np.uint32), ob) and np.array_equal(c, oc), (tag, ef)
        _, c2 = hedl.hedl_eval_batch(k, prog, 0, len(roots), flags=ef)
        assert np.array_equal(c2, oc), (tag, ef, "counts only")
    for r in eval_one:
        b1, c1 = hedl.hedl_eval_one(k, prog, r, want_bits=True)
        assert c1 == tuple(int(v) for v in oc[r]) and np.array_equal(b1.cpu().numpy().view(np.uint32), ob[r]), (tag, r)
    if device_compile:
        pd = hedl.hedl_compile_device(k, nodes, kids, roots)
        bd, cd = hedl.hedl_eval_batch(k, pd, 0, len(roots), want_bits=True)
        assert np.array_equal(bd.cpu().numpy().view(np.uint32), ob) and np.array_equal(cd, oc), (tag, "device")
        _, cdev = hedl.hedl_eval_batch(k, pd, 0, len(roots), counts_device=True)
        kk = min(16, len(roots))
        _, ti, ts = hedl.hedl_score_topk(cdev, hedl.HEDL_SCORE_F1, kk)
        oi = oscores.topk(oscores.scores(oc, oscores.F1), kk)
        assert np.array_equal(ti.cpu().numpy(), oi), (tag, "topk")
    torch.cuda.synchronize()
    print("ok", tag, flush=True)
    return k


def main():
    kb = abox.c1_kb()
    nodes, kids, roots = flatten(hyps.c1_hypotheses(kb))
    check(kb, nodes, kids, roots, (0, hedl.HEDL_EVAL_FORCE_SLICE, hedl.HEDL_EVAL_PER_NODE), "C1",
          eval_one=range(0, len(roots), 7))
    kb = abox.random_tiny_kb(7, n=40, n_roles=2, n_data=1, n_strings=2)
    rng = np.random.default_rng(7)
    trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=4) for _ in range(40)]
    check(kb, *flatten(trees), (0, hedl.HEDL_EVAL_FORCE_SLICE), "tiny strings", device_compile=False,
          eval_one=range(0, 40, 9))
    kb = abox.powerlaw_kb(20_000, 20, 2, 8.0, 2000, 0.7, 1.0, 0.02, seed=5)
    arrays = hyps.batch_arrays("c4", kb, 3000, seed=5, chunk=1000, workers=1)
    check(kb, *arrays, (0, hedl.HEDL_EVAL_NO_FUSE, hedl.HEDL_EVAL_NO_RESTRICT_U, hedl.HEDL_EVAL_PER_NODE),
          "powerlaw batch", eval_one=range(0, 3000, 500))
    # hedl_kb_set_concept_rows on a reserved slot
    import torch
    W = (kb["N"] + 31) // 32
    kb2 = dict(kb)
    kb2["concept_bits"] = np.vstack([kb["concept_bits"], np.zeros((1, W), np.uint32)])
    k = hedl.hedl_kb_load(kb2, 0)
    row = np.random.default_rng(3).integers(0, 2**32, size=(1, W), dtype=np.uint64).astype(np.uint32)
    row[0, -1] &= np.uint32((1 << (kb["N"] & 31)) - 1) if kb["N"] & 31 else np.uint32(0xffffffff)
    k.set_concept_rows(20, torch.from_numpy(row.view(np.int32)).cuda())
    kb3 = dict(kb2)
    kb3["concept_bits"] = np.vstack([kb["concept_bits"], row])
    t = [("EXISTS", 0, False, ("ATOM", 20)), ("AND", [("ATOM", 20), ("FORALL", 1, True, ("ATOM", 20))])] * 8
    nodes, kids, roots = flatten(t)
    prog = hedl.hedl_compile(k, nodes, kids, roots)
    _, c = hedl.hedl_eval_batch(k, prog, 0, len(roots))
    _, oc = setsem.evaluate(kb3, nodes, kids, roots)
    assert np.array_equal(c, oc)
    print("ok set_concept_rows", flush=True)
    print("all sanitizer cases passed", flush=True)


if __name__ == "__main__":
    main()
