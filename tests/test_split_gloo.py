"""NEXT-4: one hypothesis split across ranks by individual range, world 1/2/3 on
gloo (CPU).  The per-rank evaluator is the oracle run on the rank's PARTITION of the KB (the
assertions of its individuals + the scratch filler rows it installs), standing in for the CUDA
path; the partitioning, filler staging, segment all_gather, row installation and count
reduction are the product code in paper_2412_00802_b200/dist.py.  The summed counts must be
byte-identical to the oracle on the whole KB (results independent of the
number of devices), and every installed filler row must equal the oracle's full
row of that filler."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2412_00802_b200 import dist as hdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleSplitEvaluator:
    """eval_split's evaluator seam over the oracle and a partition dict (test infrastructure)."""

    def __init__(self, part):
        self.part = part
        self.installed = {}

    def rows(self, nodes, kids, roots):
        from oracle import setsem
        b, _ = setsem.evaluate(self.part, nodes, kids, roots, want_bits=True)
        return torch.from_numpy(b.view(np.int32).copy())

    def install(self, first, gathered, parts, part_words):
        N = self.part["N"]
        W = (N + 31) // 32
        g = gathered.cpu().numpy().view(np.uint32)                   # [parts][n][pw]
        rows = np.concatenate([g[p] for p in range(parts)], axis=1)[:, :W].copy()
        if N & 31:
            rows[:, W - 1] &= np.uint32((1 << (N & 31)) - 1)
        self.part["concept_bits"][first:first + len(rows)] = rows
        for i, r in enumerate(rows):
            self.installed[first + i] = r.copy()

    def counts(self, nodes, kids, roots):
        from oracle import setsem
        _, c = setsem.evaluate(self.part, nodes, kids, roots, want_bits=False)
        return torch.from_numpy(c.astype(np.int64))


def _cases():
    from synth import abox, hyps
    from synth.format import flatten
    out = []
    for seed in (3, 8):
        kb = abox.random_tiny_kb(seed, n=40, n_roles=2, n_data=1)
        rng = np.random.default_rng(seed)
        out.append((kb, flatten([hyps.random_tree(rng, abox.kb_shape(kb), depth=5) for _ in range(24)])))
    kb = abox.c1_kb()
    out.append((kb, flatten(hyps.c1_hypotheses(kb))))
    kb = abox.powerlaw_kb(3000, 12, 2, 6.0, 300, 0.7, 1.0, 0.05, seed=13)
    rng = np.random.default_rng(4)
    trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=5) for _ in range(30)]
    trees += [("EXISTS", 0, False, ("AND", [("ATOM", 1), ("FORALL", 1, True, ("OR", [("ATOM", 2), ("NOT", ("ATOM", 3))]))])),
              ("MIN", 2, 0, True, ("EXISTS", 1, False, ("ATOM", 4))),
              ("FORALL", 0, False, ("OR", [("EXISTS", 0, False, ("ATOM", 5)), ("DRANGE", 0, 0.5, float("inf"))]))]
    out.append((kb, flatten(trees)))
    return out


def _worker(rank, world, port, q):
    try:
        _work(rank, world, port, q)
    except BaseException as e:           # surface a rank's failure instead of a queue timeout
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        raise


def _work(rank, world, port, q):
    import torch.distributed as dist
    from oracle import setsem
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = []
    for kb, (nodes, kids, roots) in _cases():
        C = kb["concept_bits"].shape[0]
        plan = hdist.SplitPlan(nodes, kids, roots, C)
        part = hdist.partition_kb(kb, rank, world, plan.n_scratch)
        ev = OracleSplitEvaluator(part)
        counts = hdist.eval_split(plan, ev, int(kb["N"]))
        ok_rows = True
        for g, slot in plan.slot.items():            # installed filler rows == the full-KB oracle's rows
            ng = np.array([g], dtype=np.uint32)
            ob, _ = setsem.evaluate(kb, plan.nodes, plan.kids.astype(np.uint32), ng, want_bits=True)
            ok_rows &= np.array_equal(ev.installed[C + slot], ob[0])
        if rank == 0:
            _, ref = setsem.evaluate(kb, nodes, kids, roots, want_bits=False)
            res.append((counts.numpy().astype(np.uint64).tolist(), ref.tolist(), bool(ok_rows), len(plan.stages),
                        plan.n_scratch))
        else:
            assert ok_rows
    if rank == 0:
        q.put(res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_split_counts_match_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    assert not (isinstance(res, tuple) and res[0] == "error"), res
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert any(st >= 2 for _, _, _, st, _ in res), "no case exercised nested exchange stages"
    for got, ref, ok_rows, _, _ in res:
        assert got == ref
        assert ok_rows


def test_split_single_rank_and_plan():
    """World 1 (no process group): the plan's stages and rewrites alone reproduce the oracle; a
    filler below a filler gets a later stage; NOT chains over atoms need no exchange."""
    from oracle import setsem
    from synth.format import flatten
    for kb, (nodes, kids, roots) in _cases():
        C = kb["concept_bits"].shape[0]
        plan = hdist.SplitPlan(nodes, kids, roots, C)
        part = hdist.partition_kb(kb, 0, 1, plan.n_scratch)
        counts = hdist.eval_split(plan, OracleSplitEvaluator(part), int(kb["N"]))
        _, ref = setsem.evaluate(kb, nodes, kids, roots, want_bits=False)
        assert np.array_equal(counts.numpy().astype(np.uint64), ref)
    t = [("EXISTS", 0, False, ("AND", [("ATOM", 0), ("EXISTS", 1, True, ("OR", [("ATOM", 1), ("ATOM", 2)]))])),
         ("FORALL", 0, False, ("NOT", ("ATOM", 3)))]
    nodes, kids, roots = flatten(t)
    plan = hdist.SplitPlan(nodes, kids, roots, 4)
    assert plan.n_scratch == 2 and plan.stages == [1, 2]


def test_partition_kb_owns_exactly_its_assertions():
    from synth import abox
    kb = abox.random_tiny_kb(5, n=70, n_roles=2, n_data=1, n_strings=1)
    N = kb["N"]
    seen_edges = 0
    for world in (2, 3):
        for r in range(world):
            lo, hi = hdist.owned_range(N, r, world)
            p = hdist.partition_kb(kb, r, world, 3)
            assert p["concept_bits"].shape[0] == kb["concept_bits"].shape[0] + 3
            es, eo = p["edge_subj"], p["edge_obj"]
            assert (((es >= lo) & (es < hi)) | ((eo >= lo) & (eo < hi))).all()
            assert ((p["pos_ids"] >= lo) & (p["pos_ids"] < hi)).all()
            assert ((p["data_subj"] >= lo) & (p["data_subj"] < hi)).all()
            assert ((p["str_subj"] >= lo) & (p["str_subj"] < hi)).all()
            vo, blob = p["str_val_off"], p["str_bytes"]
            assert len(vo) == len(p["str_subj"]) + 1 and vo[-1] == len(blob)
            seen_edges += int((((kb["edge_subj"] >= lo) & (kb["edge_subj"] < hi))).sum())
        assert sum(len(hdist.partition_kb(kb, r, world)["pos_ids"]) for r in range(world)) == len(kb["pos_ids"])
    assert seen_edges == 2 * len(kb["edge_subj"])
