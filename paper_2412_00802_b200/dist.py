"""Multi-GPU batch dispatcher: KB replicated per GPU, hypotheses sharded.

One process per GPU (torchrun).  Every rank holds a full KB replica (the
paper's "exact copy of knowledge representation matrixes" per device,
PAPER.md:568 step 2).  The batch is cut into contiguous, cost-balanced index
ranges (static scheduling as in PAPER.md:568/578, balanced by estimated hypothesis
cost; on mixed-GPU boxes the paper's probe ratios, probe_ratios(), weight the
shares).  Each rank compiles
and evaluates only its range; the only collective is one all_gather of the
per-hypothesis count vectors (NCCL over NVLink/NVSwitch on GPUs).  Rank 0
un-pads into input order.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence, Tuple

import numpy as np

ROLE_OPS = (6, 7, 8, 9, 10)   # EXISTS..EXACT opcodes (include/hedl.h)


def root_costs(nodes: np.ndarray, child_idx: np.ndarray, roots: np.ndarray) -> np.ndarray:
    """Cheap host cost estimate per root: 1 + 16 x (role/data restrictions in its tree).

    Restrictions dominate the algorithmic bytes (a restriction
    node is ~100x a boolean node), so this tracks B(h) closely enough to
    balance shards before any rank compiles.
    """
    n = len(nodes)
    heavy = np.isin(nodes["op"], ROLE_OPS + (11, 12, 13)).astype(np.int64)
    cb = nodes["child_begin"].astype(np.int64)
    cc = nodes["child_count"].astype(np.int64)
    owner = np.repeat(np.arange(n), cc)                       # parent of each child slot
    slots = (np.repeat(cb, cc) + (np.arange(cc.sum()) - np.repeat(np.cumsum(cc) - cc, cc))
             if n else np.zeros(0, np.int64))
    kids = np.asarray(child_idx, dtype=np.int64)[slots]
    sub = heavy.copy()
    for _ in range(256):                                       # one tree level per sweep
        nxt = heavy + np.bincount(owner, weights=sub[kids], minlength=n).astype(np.int64)
        if np.array_equal(nxt, sub):
            break
        sub = nxt
    return 1 + 16 * sub[roots.astype(np.int64)]


def shard_ranges(costs: np.ndarray, world: int, weights: Optional[Sequence[float]] = None) -> list:
    """Contiguous [lo, hi) ranges, one per rank, cutting the cost prefix sums at the ranks'
    shares: equal shares by default, else proportional to `weights` (e.g. probe_ratios)."""
    n = len(costs)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * (world - 1)
    if weights is None:
        frac = np.arange(1, world, dtype=np.float64) / world
    else:
        w = np.asarray(weights, dtype=np.float64)
        assert len(w) == world and (w > 0).all(), "one positive weight per rank"
        frac = np.cumsum(w)[:-1] / w.sum()
    cum = np.cumsum(costs, dtype=np.float64)
    total = cum[-1]
    cuts = [0]
    for f in frac:
        cuts.append(int(np.searchsorted(cum, total * f, side="left")) + 1)
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def probe_ratios(kb=None, group=None, reps: int = 20, timer: Optional[Callable] = None) -> np.ndarray:
    """The paper's device-capability probe (Fig. 5 steps 3-6): every rank times a
    dummy hypothesis -- a conjunction of (up to) 5 concepts -- on its own device against the KB it
    holds; the times are all-gathered and rank r's scheduling ratio is (1/t_r) / sum(1/t).
    Computed once, then reused for every batch (static scheduling).  `timer` is a test seam
    returning this rank's probe time in seconds (the gloo tests inject one)."""
    import torch
    import torch.distributed as dist
    if timer is None:
        timer = lambda: _probe_time(kb, reps)
    t = float(timer())
    world = dist.get_world_size(group)
    dev = torch.device(f"cuda:{kb.device}") if kb is not None and dist.get_backend(group) == "nccl" else torch.device("cpu")
    buf = torch.tensor([t], dtype=torch.float64, device=dev)
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    times = np.array([float(x.item()) for x in out])
    inv = 1.0 / np.maximum(times, 1e-12)
    return inv / inv.sum()


def _probe_time(kb, reps: int) -> float:
    """Median device time of the probe hypothesis (AND of the first min(5, C) concepts).
    Its bitset is requested, so the conjunction runs over full N-bit rows (a root without
    requested bits would run on the example-projected rows and time launch latency only)."""
    import torch
    import paper_2412_00802_b200 as hedl
    c = min(5, kb.info()["C"])
    nodes = np.zeros(c + 1, dtype=hedl.HEDL_NODE_DTYPE)       # ATOM 0 .. ATOM c-1, AND(all)
    nodes["op"][:c] = 2
    nodes["arg"][:c] = np.arange(c)
    nodes["op"][c] = 4
    nodes["child_count"][c] = c
    kids = np.arange(c, dtype=np.uint32)
    prog = hedl.hedl_compile(kb, nodes, kids, np.array([c], dtype=np.uint32))
    ts = []
    with torch.cuda.device(kb.device):
        bits = torch.empty((1, max(kb.W, 1)), dtype=torch.int32, device=f"cuda:{kb.device}")
        for _ in range(reps + 3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hedl.hedl_eval_batch(kb, prog, 0, 1, counts_device=True, out_bits=bits)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1000.0)
    prog.free()
    return float(np.median(ts[3:]))


def local_arrays(nodes, child_idx, roots, lo, hi):
    """Rank-local copy of the node arrays for roots [lo, hi) when the input is post-order
    flattened trees stored root by root (every tree's nodes lie between the previous root
    and its own root, children before parents): the node range (roots[lo-1], roots[hi-1]]
    and its child slots, rebased to start at 0.  Returns None for any other layout."""
    roots = np.asarray(roots)
    if hi <= lo:
        return None
    if not np.all(np.diff(roots.astype(np.int64)) > 0):     # roots stored tree by tree, ascending
        return None
    a = int(roots[lo - 1]) + 1 if lo > 0 else 0
    b = int(roots[hi - 1]) + 1
    sub = nodes[a:b]
    r = roots[lo:hi].astype(np.int64) - a
    if len(sub) == 0 or r.min() < 0 or r.max() >= len(sub):
        return None
    cb = sub["child_begin"].astype(np.int64)
    cc = sub["child_count"].astype(np.int64)
    has = cc > 0
    k0 = int(cb[has].min()) if has.any() else 0
    k1 = int((cb + cc)[has].max()) if has.any() else 0
    kids = np.asarray(child_idx)[k0:k1].astype(np.int64) - a
    if len(kids) and (kids.min() < 0 or kids.max() >= len(sub)):
        return None
    out = sub.copy()
    out["child_begin"] = np.where(has, cb - k0, 0).astype(np.uint32)
    return out, kids.astype(np.uint32), r.astype(np.uint32)


def gather_counts(local_counts, n_total: int, ranges, group=None, device=None):
    """all_gather the padded per-rank count blocks; every rank gets counts[n_total][4] (input order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    pad = max(hi - lo for lo, hi in ranges) if ranges else 0
    pad = max(pad, 1)
    buf = torch.zeros((pad, 4), dtype=torch.int64, device=device)
    n_loc = local_counts.shape[0]
    if n_loc:
        buf[:n_loc].copy_(local_counts)
    out = torch.empty((world * pad, 4), dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, buf, group=group)
    parts = [out[r * pad:r * pad + (hi - lo)] for r, (lo, hi) in enumerate(ranges)]
    res = torch.cat(parts, 0) if parts else out[:0]
    assert res.shape[0] == n_total
    return res


def eval_batch_sharded(kb, nodes: np.ndarray, child_idx: np.ndarray, roots: np.ndarray,
                       flags: int = 0, group=None,
                       evaluator: Optional[Callable] = None,
                       weights: Optional[Sequence[float]] = None) -> Tuple["object", dict]:
    """Evaluate the batch across the ranks of `group`; returns (counts[n][4] int64 tensor, info).

    `kb` is this rank's replica (a paper_2412_00802_b200.KB).  `evaluator`
    is a test seam (the CPU gloo tests inject one); by default each rank runs
    hedl_compile + hedl_eval_batch (device counts) through the C ABI.
    """
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    costs = root_costs(nodes, child_idx, roots)
    ranges = shard_ranges(costs, world, weights)
    lo, hi = ranges[rank]
    if evaluator is None:
        import paper_2412_00802_b200 as hedl
        dev = torch.device(f"cuda:{kb.device}")
        if hi > lo:
            prog = hedl.hedl_compile(kb, nodes, child_idx, roots[lo:hi], flags)
            _, local = hedl.hedl_eval_batch(kb, prog, 0, hi - lo, counts_device=True)
        else:
            local = torch.zeros((0, 4), dtype=torch.int64, device=dev)
    else:
        dev = torch.device("cpu")
        local = evaluator(nodes, child_idx, roots[lo:hi])
    counts = gather_counts(local, len(roots), ranges, group=group, device=dev)
    return counts, {"ranges": ranges, "rank": rank, "world": world}
