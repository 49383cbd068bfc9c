"""Host timeline of bench.py's double-buffered e2e loop (C4): per iteration, the host time
spent issuing the H2D, in hedl_compile_device, in hedl_eval_batch, and in program frees."""
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
    sys.argv = [sys.argv[0]]
    args = bench.parse()
    kb_np, nodes, kids, roots = bench.c4_inputs(args, 1)
    kb = hedl.hedl_kb_load(kb_np, 0)
    dev = torch.device("cuda:0")
    n_loc = len(roots)
    pins = [torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1)).pin_memory()
            for a in (nodes, np.asarray(kids, np.uint32), np.asarray(roots, np.uint32))]
    s_eval = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]
    s_comp = torch.cuda.Stream(device=dev, priority=-1)
    s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    dbuf = [tuple(torch.empty_like(t, device=dev) for t in pins) for _ in range(2)]
    cdev = [torch.empty((n_loc, 4), dtype=torch.int64, device=dev) for _ in range(2)]
    chost = [torch.empty((n_loc, 4), dtype=torch.int64).pin_memory() for _ in range(2)]
    h2d_done, comp_done, eval_done, d2h_done = ([torch.cuda.Event(), torch.cuda.Event()] for _ in range(4))
    mode = os.environ.get("PIPE_MODE", "pipe")

    def issue_h2d(k):
        b = k & 1
        with torch.cuda.stream(s_h2d):
            s_h2d.wait_event(comp_done[b])
            for dst, src in zip(dbuf[b], pins):
                dst.copy_(src, non_blocking=True)
            h2d_done[b].record(s_h2d)

    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        issue_h2d(0)
        progs, rows = [], []
        n = 8
        for k in range(n):
            b = k & 1
            ta = time.perf_counter()
            if k + 1 < n:
                issue_h2d(k + 1)
            tb = time.perf_counter()
            s_comp.wait_event(h2d_done[b])
            p2 = hedl.hedl_compile_device(kb, *dbuf[b], n_nodes=len(nodes), n_kids=len(kids), n_roots=n_loc, stream=s_comp)
            comp_done[b].record(s_comp)
            tc = time.perf_counter()
            s_eval[b].wait_event(comp_done[b])
            s_eval[b].wait_event(d2h_done[b])
            hedl.hedl_eval_batch(kb, p2, 0, n_loc, counts_device=True, out_counts=cdev[b], stream=s_eval[b])
            eval_done[b].record(s_eval[b])
            td = time.perf_counter()
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(eval_done[b])
                chost[b].copy_(cdev[b], non_blocking=True)
                d2h_done[b].record(s_d2h)
            progs.append(p2)
            if len(progs) > 2:
                progs.pop(0).free()
            te = time.perf_counter()
            if mode == "seq":
                torch.cuda.synchronize()
            ms = torch.cuda.memory_stats(dev)
            rows.append([1000 * (x - t0) for x in (ta, tb, tc, td, te)] +
                        [ms.get("num_alloc_retries", 0), ms.get("num_device_alloc", 0), ms.get("num_device_free", 0),
                         torch.cuda.memory_reserved(dev) / 2**30] + list(hedl.alloc_counters()))
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        for q in progs:
            q.free()
        print(f"rep {rep} mode {mode}: {1000 * el / n:.2f} ms/step")
        for k, r in enumerate(rows):
            print(f"  it {k}: start {r[0]:8.2f}  h2d-issue {r[1] - r[0]:6.2f}  compile {r[2] - r[1]:6.2f}  "
                  f"eval {r[3] - r[2]:6.2f}  d2h+free {r[4] - r[3]:6.2f}  retries {r[5]} cudaMalloc {r[6]} cudaFree {r[7]} "
                  f"reserved {r[8]:.1f} GiB  hedl allocs {r[9:]}")


if __name__ == "__main__":
    main()
