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


# ---------------------------------------------------------------------------------------------
# NEXT-4: ONE hypothesis (or batch) split across ranks by individual range (
# PAPER.md:563-578 multi-device scheduling, "GPUs have fixed memory sizes, which
# limits certain GPUs to certain dataset sizes").
#
# Rank r owns the words [r*pw, (r+1)*pw) of every row (pw = ceil(W / G)), i.e. individuals
# 32*r*pw .. 32*(r+1)*pw - 1, and holds only the assertions it needs for them: role pairs whose
# subject (rows of r) or object (rows of r^-) it owns, data / string assertions of its
# subjects, its own examples.  Concept rows are replicated (C x W bits), plus one reserved
# "scratch" concept per restriction filler that must be complete.
#
# Every node is evaluated for the owned individuals only -- booleans and ranges are word-local,
# a restriction at an owned x reads all of x's pairs (they are all on the rank) -- except that a
# restriction reads its filler at ANY neighbour.  So each non-atomic filler is an exchange
# point: the ranks evaluate it (their segments are correct), all_gather the segments, and
# install the complete row as its scratch concept (hedl_kb_set_concept_rows), innermost
# fillers first.  The roots are then evaluated against the owned examples only and the four
# counts summed across ranks (an owned-example count per rank: tp = sum tp_r, fn = |P| - tp).
# ---------------------------------------------------------------------------------------------
OP_TOP, OP_BOTTOM, OP_ATOM, OP_NOT = 0, 1, 2, 3


def split_words(W: int, world: int) -> int:
    """Words per rank segment (the last segment may be short)."""
    return max(1, -(-W // max(1, world)))


def owned_range(N: int, rank: int, world: int):
    """[lo, hi) individuals owned by `rank`."""
    W = (N + 31) // 32
    pw = split_words(W, world)
    return min(N, 32 * pw * rank), min(N, 32 * pw * (rank + 1))


class SplitPlan:
    """Exchange points of a node batch: the restriction fillers (NOT chains stripped) that are
    not atoms / TOP / BOTTOM, each with a scratch concept slot and a stage (1 + the deepest
    stage of the fillers nested in it); slots are numbered stage by stage.  `arrays(s)` gives
    the batch with every filler of a stage < s replaced by its scratch atom (s = None: all)."""

    def __init__(self, nodes: np.ndarray, child_idx: np.ndarray, roots: np.ndarray, n_concepts: int):
        self.nodes, self.kids, self.roots = nodes, np.asarray(child_idx, dtype=np.int64), np.asarray(roots)
        self.C0 = int(n_concepts)
        op = nodes["op"].astype(np.int64)
        cb = nodes["child_begin"].astype(np.int64)
        cc = nodes["child_count"].astype(np.int64)
        n = len(nodes)
        owner = np.repeat(np.arange(n), cc)                              # parent of each child slot
        slots = (np.repeat(cb, cc) + (np.arange(cc.sum()) - np.repeat(np.cumsum(cc) - cc, cc))
                 if n else np.zeros(0, np.int64))
        kid = self.kids[slots]
        reach = np.zeros(n, dtype=bool)                                  # reachable from the roots
        reach[self.roots.astype(np.int64)] = True
        while True:
            nxt = reach.copy()
            nxt[kid[reach[owner]]] = True
            if np.array_equal(nxt, reach):
                break
            reach = nxt
        self.reach = reach

        def strip(i):
            while op[i] == OP_NOT:
                i = int(self.kids[cb[i]])
            return i

        isg = np.zeros(n, dtype=bool)
        for i in np.nonzero(np.isin(op, ROLE_OPS) & reach)[0]:
            g = strip(int(self.kids[cb[i]]))
            if op[g] not in (OP_TOP, OP_BOTTOM, OP_ATOM):
                isg[g] = True
        # stage(g) = 1 + the deepest stage among the fillers below g (relaxation, one level a sweep)
        below = np.zeros(n, dtype=np.int64)
        while True:
            contrib = np.where(isg[kid], below[kid] + 1, below[kid])
            nb = np.zeros(n, dtype=np.int64)
            np.maximum.at(nb, owner, contrib)
            if np.array_equal(nb, below):
                break
            below = nb
        gather = {int(g): int(below[g]) + 1 for g in np.nonzero(isg)[0]}
        self.gather = gather
        self.stages = sorted(set(gather.values()))
        order = sorted(gather, key=lambda g: (gather[g], g))
        self.slot = {g: k for k, g in enumerate(order)}
        self.n_scratch = len(order)
        self.items = {s: [g for g in order if gather[g] == s] for s in self.stages}
        # appended ATOM nodes, one per gather node (its scratch concept)
        ext = np.zeros(self.n_scratch, dtype=nodes.dtype)
        ext["op"] = OP_ATOM
        ext["arg"] = [self.C0 + self.slot[g] for g in order]
        self.ext_nodes = np.concatenate([nodes, ext]) if self.n_scratch else nodes
        if hasattr(nodes, "patterns") and self.ext_nodes is not nodes:   # the string-pattern table
            self.ext_nodes = self.ext_nodes.view(type(nodes))
            self.ext_nodes.patterns = nodes.patterns
        self.atom_of = np.arange(n + self.n_scratch, dtype=np.int64)
        for g in order:
            self.atom_of[g] = n + self.slot[g]

    def arrays(self, stage=None):
        """(nodes, child_idx, roots) of stage `stage` (its fillers as roots) or, with None, of the
        final pass (the batch roots), every filler of an earlier stage read as its scratch atom."""
        repl = np.zeros(len(self.atom_of), dtype=bool)
        for g, s in self.gather.items():
            if stage is None or s < stage:
                repl[g] = True
        kids = np.where(repl[self.kids], self.atom_of[self.kids], self.kids).astype(np.uint32)
        if stage is None:
            roots = np.where(repl[self.roots.astype(np.int64)], self.atom_of[self.roots.astype(np.int64)],
                             self.roots).astype(np.uint32)
        else:
            roots = np.array(self.items[stage], dtype=np.uint32)
        return self.ext_nodes, kids, roots

    def first_slot(self, stage) -> int:
        return self.slot[self.items[stage][0]]


def partition_kb(kb: dict, rank: int, world: int, n_scratch: int = 0) -> dict:
    """The KB arrays rank `rank` holds: every concept row (+ n_scratch zero rows for the
    fillers), role pairs with an owned subject or object, data / string assertions and examples
    of owned individuals.  Ids stay global."""
    N = int(kb["N"])
    lo, hi = owned_range(N, rank, world)
    own = lambda ids: (ids >= lo) & (ids < hi)
    W = (N + 31) // 32
    cb = np.asarray(kb["concept_bits"], dtype=np.uint32).reshape(-1, W) if W else \
        np.zeros((len(kb["concept_bits"]), 0), np.uint32)
    out = {"N": N, "concept_bits": np.vstack([cb, np.zeros((n_scratch, W), np.uint32)]) if n_scratch else cb}
    off = np.asarray(kb["role_edge_off"], dtype=np.uint64)
    es, eo = np.asarray(kb["edge_subj"], np.uint32), np.asarray(kb["edge_obj"], np.uint32)
    keep = own(es) | own(eo)
    cnt = [int(keep[int(off[r]):int(off[r + 1])].sum()) for r in range(len(off) - 1)]
    out["role_edge_off"] = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64)
    out["edge_subj"], out["edge_obj"] = es[keep], eo[keep]
    doff = np.asarray(kb["data_off"], dtype=np.uint64)
    ds = np.asarray(kb["data_subj"], np.uint32)
    dk = own(ds)
    dcnt = [int(dk[int(doff[d]):int(doff[d + 1])].sum()) for d in range(len(doff) - 1)]
    out["data_off"] = np.concatenate([[0], np.cumsum(dcnt)]).astype(np.uint64)
    out["data_subj"], out["data_val"] = ds[dk], np.asarray(kb["data_val"], np.float32)[dk]
    p, q = np.asarray(kb["pos_ids"], np.uint32), np.asarray(kb["neg_ids"], np.uint32)
    out["pos_ids"], out["neg_ids"] = p[own(p)], q[own(q)]
    if "str_off" in kb:
        soff = np.asarray(kb["str_off"], np.uint64)
        ss = np.asarray(kb["str_subj"], np.uint32)
        vo = np.asarray(kb["str_val_off"], np.uint64)
        blob = np.asarray(kb["str_bytes"], np.uint8)
        sk = own(ss)
        scnt = [int(sk[int(soff[s]):int(soff[s + 1])].sum()) for s in range(len(soff) - 1)]
        idx = np.nonzero(sk)[0]
        lens = (vo[idx + 1] - vo[idx]).astype(np.int64)
        starts = vo[idx].astype(np.int64)
        pos = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(lens.sum())
        out["str_off"] = np.concatenate([[0], np.cumsum(scnt)]).astype(np.uint64)
        out["str_subj"] = ss[sk]
        out["str_val_off"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        out["str_bytes"] = blob[pos] if len(pos) else np.zeros(0, np.uint8)
    return out


class GpuSplitEvaluator:
    """The per-rank evaluation of eval_split through the C ABI (kb = the rank's partition,
    loaded as a paper_2412_00802_b200.KB)."""

    def __init__(self, kb, flags: int = 0):
        self.kb, self.flags = kb, flags

    def rows(self, nodes, kids, roots):
        import paper_2412_00802_b200 as hedl
        prog = hedl.hedl_compile(self.kb, nodes, kids, roots, self.flags)
        bits, _ = hedl.hedl_eval_batch(self.kb, prog, 0, len(roots), want_bits=True)
        prog.free()
        return bits                                     # CUDA int32 [n][W]

    def install(self, first, gathered, parts, part_words):
        self.kb.set_concept_rows(first, gathered, parts, part_words)

    def counts(self, nodes, kids, roots):
        import paper_2412_00802_b200 as hedl
        prog = hedl.hedl_compile(self.kb, nodes, kids, roots, self.flags)
        _, c = hedl.hedl_eval_batch(self.kb, prog, 0, len(roots), counts_device=True)
        prog.free()
        return c                                        # CUDA int64 [n][4]


def eval_split(plan: SplitPlan, evaluator, N: int, group=None, device=None):
    """Evaluate plan's roots with the individuals split across the ranks of `group` (every rank
    calls it with the same plan and its own evaluator).  Returns counts[n_roots][4] (int64
    tensor, input order) on every rank.  `evaluator` has rows(nodes, kids, roots) -> [n][W]
    rows correct on the owned words, install(first_slot, rows[parts][n][part_words], parts,
    part_words) and counts(nodes, kids, roots) -> [n][4] over the owned examples
    (GpuSplitEvaluator on GPUs; the CPU gloo tests inject one built on the oracle)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    W = (N + 31) // 32
    pw = split_words(W, world)
    for s in plan.stages:
        nodes, kids, roots = plan.arrays(s)
        rows = evaluator.rows(nodes, kids, roots)
        rows = torch.as_tensor(rows).view(torch.int32) if not isinstance(rows, torch.Tensor) else rows.view(torch.int32)
        n = rows.shape[0]
        seg = torch.zeros((n, pw), dtype=torch.int32, device=rows.device)
        a, b = min(W, rank * pw), min(W, (rank + 1) * pw)
        if b > a:
            seg[:, :b - a] = rows[:, a:b]
        if world > 1:
            dev = device if device is not None else rows.device
            out = torch.empty((world * n, pw), dtype=torch.int32, device=dev)
            dist.all_gather_into_tensor(out, seg.to(dev), group=group)
            gathered = out.view(world, n, pw)
        else:
            gathered = seg.view(1, n, pw)
        evaluator.install(plan.C0 + plan.first_slot(s), gathered.to(rows.device).contiguous(), world, pw)
    nodes, kids, roots = plan.arrays(None)
    c = evaluator.counts(nodes, kids, roots)
    c = torch.as_tensor(np.asarray(c).view(np.int64)) if not isinstance(c, torch.Tensor) else c
    if world > 1:
        dev = device if device is not None else c.device
        c2 = c.to(dev).clone()
        dist.all_reduce(c2, op=dist.ReduceOp.SUM, group=group)
        c = c2
    return c
