"""NEXT-4 on the GPU: hedl_kb_set_concept_rows and the individual-range split of one hypothesis
batch (paper_2412_00802_b200/dist.py eval_split), through the C ABI, against
the oracle on the whole KB (bit-exact counts)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import setsem
from paper_2412_00802_b200 import dist as hdist
from synth import abox, hyps
from synth.format import flatten
from test_gpu_parity import _hedl

pytestmark = pytest.mark.gpu


def _kb():
    return abox.powerlaw_kb(120_000, 50, 2, 8.0, 3000, 0.7, 1.0, 0.01, seed=21)


def _trees(kb, n=40, seed=4):
    rng = np.random.default_rng(seed)
    shape = abox.kb_shape(kb)
    t = [hyps.random_tree(rng, shape, depth=5) for _ in range(n)]
    t += hyps.c3_hypotheses()
    return t


def test_set_concept_rows_updates_projections():
    """A row installed into a reserved concept slot is read like a loaded concept by every path:
    full-row packs, example-row (EX) packs over U rows, per-node kernels, example-projected
    booleans -- the oracle sees a KB whose concept row is that row."""
    hedl = _hedl()
    kb = _kb()
    N, W = kb["N"], (kb["N"] + 31) // 32
    C = kb["concept_bits"].shape[0]
    kb2 = dict(kb)
    kb2["concept_bits"] = np.vstack([kb["concept_bits"], np.zeros((2, W), np.uint32)])
    k = hedl.hedl_kb_load(kb2, 0)
    rng = np.random.default_rng(1)
    rows = rng.integers(0, 2**32, size=(2, W), dtype=np.uint64).astype(np.uint32)
    rows[:, -1] &= np.uint32((1 << (N & 31)) - 1) if N & 31 else np.uint32(0xffffffff)
    k.set_concept_rows(C, torch.from_numpy(rows.view(np.int32)).cuda())
    kb3 = dict(kb2)
    kb3["concept_bits"] = np.vstack([kb["concept_bits"], rows])
    A = lambda i: ("ATOM", i)
    trees = []
    for r in range(2):
        for inv in (False, True):
            for c in (C, C + 1):
                trees += [("EXISTS", r, inv, A(c)), ("FORALL", r, inv, ("NOT", A(c))), ("MIN", 3, r, inv, A(c)),
                          ("AND", [A(c), ("EXISTS", r, inv, ("OR", [A(c), A(1)]))]), ("OR", [("NOT", A(c)), A(0)])]
    trees = trees * 3                                 # enough restrictions per group for the packs
    nodes, kids, roots = flatten(trees)
    prog = hedl.hedl_compile(k, nodes, kids, roots)
    _, c = hedl.hedl_eval_batch(k, prog, 0, len(roots))
    b, cb = hedl.hedl_eval_batch(k, prog, 0, 40, want_bits=True)
    ob, oc = setsem.evaluate(kb3, nodes, kids, roots, threads=os.cpu_count())
    assert np.array_equal(c, oc)
    assert np.array_equal(b.cpu().numpy().view(np.uint32), ob[:40]) and np.array_equal(cb, oc[:40])


def test_split_world1_in_process():
    hedl = _hedl()
    kb = _kb()
    nodes, kids, roots = flatten(_trees(kb))
    C = kb["concept_bits"].shape[0]
    plan = hdist.SplitPlan(nodes, kids, roots, C)
    assert len(plan.stages) >= 2
    k = hedl.hedl_kb_load(hdist.partition_kb(kb, 0, 1, plan.n_scratch), 0)
    counts = hdist.eval_split(plan, hdist.GpuSplitEvaluator(k), kb["N"])
    _, ref = setsem.evaluate(kb, nodes, kids, roots, threads=os.cpu_count())
    assert np.array_equal(counts.cpu().numpy().view(np.uint64), ref)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        import paper_2412_00802_b200 as hedl
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        kb = _kb()
        nodes, kids, roots = flatten(_trees(kb))
        plan = hdist.SplitPlan(nodes, kids, roots, kb["concept_bits"].shape[0])
        k = hedl.hedl_kb_load(hdist.partition_kb(kb, rank, world, plan.n_scratch), 0)
        counts = hdist.eval_split(plan, hdist.GpuSplitEvaluator(k), kb["N"], device=torch.device("cpu"))
        if rank == 0:
            q.put(("ok", counts.cpu().numpy().view(np.uint64).tolist()))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException:
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_split_multiprocess_one_gpu(world):
    """World 2 / 3: the ranks are processes sharing cuda:0 (this box has one GPU), collectives on
    gloo; each rank holds only its partition of the assertions."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=900)
    for p in procs:
        p.join(120)
    assert res[0] == "ok", res
    kb = _kb()
    nodes, kids, roots = flatten(_trees(kb))
    _, ref = setsem.evaluate(kb, nodes, kids, roots, threads=os.cpu_count())
    assert np.array_equal(np.array(res[1], dtype=np.uint64), ref)
    for p in procs:
        assert p.exitcode == 0
