"""Multi-GPU batch dispatcher: KB replicated per GPU, hypotheses sharded.

One process per GPU (torchrun).  Every rank holds a full KB replica (the
paper's "exact copy of knowledge representation matrixes" per device,
PAPER.md:568 step 2).  The batch is cut into contiguous, cost-balanced index
ranges (static scheduling as in PAPER.md:568/578, with estimated hypothesis
cost replacing device speed: the B200s are identical).  Each rank compiles
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


def shard_ranges(costs: np.ndarray, world: int) -> list:
    """Contiguous [lo, hi) ranges with near-equal cost prefix sums (one per rank)."""
    n = len(costs)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * (world - 1)
    cum = np.cumsum(costs, dtype=np.float64)
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")) + 1)
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def local_arrays(nodes, child_idx, roots, lo, hi):
    """Rank-local copy of the node arrays for roots [lo, hi) when the input is post-order
    flattened trees stored root by root (every tree's nodes lie between the previous root
    and its own root, children before parents): the node range (roots[lo-1], roots[hi-1]]
    and its child slots, rebased to start at 0.  Returns None for any other layout."""
    roots = np.asarray(roots)
    if hi <= lo:
        return None
    a = int(roots[lo - 1]) + 1 if lo > 0 else 0
    b = int(roots[hi - 1]) + 1
    if lo > 0 and not np.all(np.diff(roots.astype(np.int64)) > 0):
        return None
    sub = nodes[a:b]
    r = roots[lo:hi].astype(np.int64) - a
    if len(sub) == 0 or r.min() < 0:
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


def subset_arrays(nodes, child_idx, roots, lo, hi):
    """The node arrays restricted to roots [lo, hi) (all nodes kept; roots sliced)."""
    return nodes, child_idx, roots[lo:hi]


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
                       evaluator: Optional[Callable] = None) -> Tuple["object", dict]:
    """Evaluate the batch across the ranks of `group`; returns (counts[n][4] int64 tensor, info).

    `kb` is this rank's replica (a paper_2412_00802_b200.KB).  `evaluator`
    is a test seam (the CPU gloo tests inject one); by default each rank runs
    hedl_compile + hedl_eval_batch (device counts) through the C ABI.
    """
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    costs = root_costs(nodes, child_idx, roots)
    ranges = shard_ranges(costs, world)
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
