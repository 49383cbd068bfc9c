"""Breakdown of bench.py's e2e / learner step (host wall time per phase, synchronised)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2412_00802_b200 as hedl  # noqa: E402


def main():
    args = bench.parse()
    kb_np, nodes, kids, roots = bench.c4_inputs(args, 1)
    kb = hedl.hedl_kb_load(kb_np, 0)
    dev = torch.device("cuda:0")
    nodes_pin = torch.from_numpy(np.ascontiguousarray(nodes).view(np.uint8).reshape(-1)).pin_memory()
    kids_pin = torch.from_numpy(np.ascontiguousarray(kids, dtype=np.uint32).view(np.uint8)).pin_memory()
    roots_pin = torch.from_numpy(np.ascontiguousarray(roots, dtype=np.uint32).view(np.uint8)).pin_memory()
    nd, kd, rd = (torch.empty_like(t, device=dev) for t in (nodes_pin, kids_pin, roots_pin))
    for it in range(int(os.environ.get("E2E_ITERS", "8"))):
        T = {}
        torch.cuda.synchronize()
        t = time.perf_counter()

        def mark(name):
            nonlocal t
            torch.cuda.synchronize()
            now = time.perf_counter()
            T[name] = round(1000 * (now - t), 2)
            t = now
        nd.copy_(nodes_pin, non_blocking=True)
        kd.copy_(kids_pin, non_blocking=True)
        rd.copy_(roots_pin, non_blocking=True)
        mark("h2d")
        p = hedl.hedl_compile_device(kb, nd, kd, rd, n_nodes=len(nodes), n_kids=len(kids), n_roots=len(roots))
        mark("compile")
        _, c = hedl.hedl_eval_batch(kb, p, 0, len(roots), counts_device=True)
        mark("plan+eval")
        _, c = hedl.hedl_eval_batch(kb, p, 0, len(roots), counts_device=True)
        mark("eval (cached plan)")
        _, ti, ts = hedl.hedl_score_topk(c, hedl.HEDL_SCORE_F1, 1000, want_scores=False)
        mark("score+topk")
        ti.cpu()
        mark("d2h topk")
        ch = c.cpu()
        mark("d2h counts")
        p.free()
        mark("free")
        print(it, T, flush=True)


if __name__ == "__main__":
    main()
