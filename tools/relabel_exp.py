"""Experiment: does relabelling individuals for locality speed up the C4
sweep?  Counts do not depend on the labels, so the same batch runs on the KB as generated and
on relabelled copies; counts must be identical, and the per-class kernel times are compared.

  python tools/relabel_exp.py [--orders none,degree,bfs] [--steps 5]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def degree_order(kb):
    """new label of each individual: rank by total degree (in + out over every role), descending"""
    N = kb["N"]
    deg = np.bincount(kb["edge_subj"], minlength=N) + np.bincount(kb["edge_obj"], minlength=N)
    order = np.argsort(-deg, kind="stable")          # order[new] = old
    return order


def bfs_order(kb):
    """degree-descending seeds, BFS over the undirected role graph, neighbours by degree"""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import breadth_first_order
    N = kb["N"]
    s, o = kb["edge_subj"].astype(np.int64), kb["edge_obj"].astype(np.int64)
    A = sp.csr_matrix((np.ones(2 * len(s), np.int8), (np.concatenate([s, o]), np.concatenate([o, s]))), shape=(N, N))
    deg = np.diff(A.indptr)
    by_deg = np.argsort(-deg, kind="stable")
    comp = breadth_first_order(A, int(by_deg[0]), directed=False, return_predecessors=False)
    seen = np.zeros(N, bool)
    seen[comp] = True
    return np.concatenate([comp, by_deg[~seen[by_deg]]])   # the giant component, then the rest by degree


def permute_bits(rows, N, order):
    W = rows.shape[1]
    bits = np.unpackbits(rows.view(np.uint8).reshape(rows.shape[0], -1), axis=1, bitorder="little")[:, :N]
    nb = bits[:, order]
    out = np.zeros((rows.shape[0], W * 32), np.uint8)
    out[:, :N] = nb
    return np.packbits(out, axis=1, bitorder="little").view(np.uint32).reshape(rows.shape[0], W)


def relabel(kb, order):
    N = kb["N"]
    new_of = np.empty(N, np.uint32)
    new_of[order] = np.arange(N, dtype=np.uint32)
    k = dict(kb)
    k["concept_bits"] = permute_bits(kb["concept_bits"], N, order)
    k["edge_subj"] = new_of[kb["edge_subj"]]
    k["edge_obj"] = new_of[kb["edge_obj"]]
    k["data_subj"] = new_of[kb["data_subj"]]
    k["pos_ids"] = np.sort(new_of[kb["pos_ids"]])
    k["neg_ids"] = np.sort(new_of[kb["neg_ids"]])
    # data assertions must stay grouped by property; within a property any order is accepted
    return k


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", default="none,degree,bfs")
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    import torch
    import bench
    import paper_2412_00802_b200 as hedl
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    kb0 = bench.workload_kb("c4", args)
    nodes, kids, roots = bench.rank_hyps("c4", kb0, 1_000_000, 0, args)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ref = None
    for name in a.orders.split(","):
        t0 = time.time()
        kb = kb0 if name == "none" else relabel(kb0, degree_order(kb0) if name == "degree" else bfs_order(kb0))
        tp = time.time() - t0
        k = hedl.hedl_kb_load(kb, 0)
        prog = hedl.hedl_compile(k, nodes, kids, roots)
        out = torch.empty((len(roots), 4), dtype=torch.int64, device="cuda")
        for _ in range(3):
            hedl.hedl_eval_batch(k, prog, 0, len(roots), counts_device=True, out_counts=out)
        times = []
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            hedl.hedl_eval_batch(k, prog, 0, len(roots), counts_device=True, out_counts=out)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        c = out.cpu().numpy()
        same = ref is None or np.array_equal(c, ref)
        ref = c if ref is None else ref
        hedl.prof_reset()
        hedl.prof_enable(True)
        for _ in range(2):
            flush.zero_()
            hedl.hedl_eval_batch(k, prog, 0, len(roots), counts_device=True, out_counts=out)
        torch.cuda.synchronize()
        hedl.prof_enable(False)
        prof = hedl.prof_read()
        cls = "  ".join(f"{p['name']} {p['total_ms'] / 2:.3f}" for p in sorted(prof, key=lambda p: -p["total_ms"])[:7])
        print(f"{name:7s} relabel {tp:5.1f}s  step {np.median(times):.3f} ms  counts_equal {same}  | {cls}", flush=True)
        del prog, k


if __name__ == "__main__":
    main()
