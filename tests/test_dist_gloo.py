"""Multi-process (world_size 2 and 3, gloo on CPU) coverage of the sharded dispatcher's host logic.

The per-rank evaluator is injected (the oracle stands in for the CUDA path,
which needs a GPU); sharding, padding, all_gather and un-padding are the
product code in paper_2412_00802_b200/dist.py.  Results must be independent
of the number of ranks and in input order.
"""
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


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import setsem
    from synth import abox, hyps
    from synth.format import flatten
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kb = abox.random_tiny_kb(3, n=40, n_roles=2, n_data=1)
    rng = np.random.default_rng(5)
    trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=4) for _ in range(37)]
    nodes, kids, roots = flatten(trees)
    okb = setsem.OracleKB(kb)

    def evaluator(n, k, r):
        _, c = okb.evaluate(n, k, r, want_bits=False)
        return torch.from_numpy(c.astype(np.int64))

    counts, info = hdist.eval_batch_sharded(None, nodes, kids, roots, evaluator=evaluator)
    if rank == 0:
        _, ref = okb.evaluate(nodes, kids, roots, want_bits=False)
        q.put((counts.numpy().tolist(), ref.astype(np.int64).tolist(), info["ranges"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_counts_match_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        got, ref, ranges = q.get(timeout=180)
    except Exception:
        for p in procs:
            p.kill()
        raise
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert got == ref
    assert ranges[0][0] == 0 and ranges[-1][1] == 37
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def test_shard_ranges_balanced():
    rng = np.random.default_rng(0)
    costs = rng.integers(1, 100, 10_000)
    for world in (1, 2, 4, 8):
        rs = hdist.shard_ranges(costs, world)
        assert rs[0][0] == 0 and rs[-1][1] == len(costs) and len(rs) == world
        loads = [costs[a:b].sum() for a, b in rs]
        assert max(loads) <= costs.sum() / world + costs.max()
    assert hdist.shard_ranges(np.ones(3), 8)[-1] == (3, 3)


def test_root_costs_counts_restrictions():
    from synth.format import flatten
    trees = [("ATOM", 0), ("EXISTS", 0, False, ("AND", [("ATOM", 1), ("FORALL", 1, True, ("TOP",))])),
             ("DRANGE", 0, 0.0, 1.0)]
    nodes, kids, roots = flatten(trees)
    assert hdist.root_costs(nodes, kids, roots).tolist() == [1, 33, 17]


def test_local_arrays_rebased_equal_results():
    """Rank-local rebased node arrays (post-order batches) give the oracle's counts for that range."""
    from oracle import setsem
    from synth import abox, hyps
    from synth.format import flatten
    kb = abox.random_tiny_kb(11, n=40, n_roles=2, n_data=1, n_strings=0)
    rng = np.random.default_rng(2)
    trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=4) for _ in range(50)]
    nodes, kids, roots = flatten(trees)
    _, ref = setsem.evaluate(kb, nodes, kids, roots, want_bits=False)
    for lo, hi in ((0, 50), (0, 1), (7, 31), (49, 50)):
        loc = hdist.local_arrays(nodes, kids, roots, lo, hi)
        assert loc is not None
        n2, k2, r2 = loc
        assert len(n2) <= len(nodes)
        _, c = setsem.evaluate(kb, n2, k2, r2, want_bits=False)
        assert (c == ref[lo:hi]).all(), (lo, hi)
    shared = flatten(trees, share=True)                  # DAG input: later trees reuse earlier nodes
    loc = hdist.local_arrays(*shared, 3, 9)
    if loc is not None:                                  # only when the range is self-contained
        _, c = setsem.evaluate(kb, *loc, want_bits=False)
        assert (c == ref[3:9]).all()


def test_local_arrays_rejects_unsorted_roots():
    """Roots out of tree order (also for a range starting at 0) are not a post-order batch:
    local_arrays returns None instead of a slice that cuts off later roots."""
    from synth import abox, hyps
    from synth.format import flatten
    kb = abox.random_tiny_kb(12, n=40, n_roles=2, n_data=1, n_strings=0)
    rng = np.random.default_rng(3)
    nodes, kids, roots = flatten([hyps.random_tree(rng, abox.kb_shape(kb), depth=3) for _ in range(6)])
    perm = roots[[0, 5, 1, 2, 3, 4]]
    assert hdist.local_arrays(nodes, kids, perm, 0, 3) is None
    assert hdist.local_arrays(nodes, kids, perm, 2, 5) is None
    assert hdist.local_arrays(nodes, kids, roots, 0, 3) is not None


def _probe_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r's device is (r+1)x slower: ratios 1/(r+1) normalised
    ratios = hdist.probe_ratios(timer=lambda: 0.001 * (rank + 1))
    q.put((rank, ratios.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_probe_ratios_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_probe_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    inv = np.array([1.0 / (r + 1) for r in range(world)])
    for _, ratios in got:                                   # every rank gets the same ratios
        assert np.allclose(ratios, inv / inv.sum())


def test_weighted_shard_ranges():
    costs = np.ones(1000)
    r = hdist.shard_ranges(costs, 3, weights=[0.5, 0.25, 0.25])
    assert r == [(0, 501), (501, 751), (751, 1000)] or abs(r[0][1] - 500) <= 1
    assert r[0][0] == 0 and r[-1][1] == 1000 and all(a[1] == b[0] for a, b in zip(r, r[1:]))
    sizes = [b - a for a, b in r]
    assert abs(sizes[0] - 500) <= 2 and abs(sizes[1] - 250) <= 2


def test_bench_multirank_dry_run(tmp_path):
    """bench.py's multi-rank path under torchrun (world 2, gloo, no GPU): each rank builds only its
    own beams of the batch (their node arrays differ), caches are written race-free, and the count
    all_gather returns every root in global order."""
    import json
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
           "--dry-run", "--gpus", "2", "--n-hyps", "2000", "--n-individuals", "20000", "--cache", str(tmp_path)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["dry_run"] and line["world"] == 2 and line["gather_in_order"]
    assert line["node_digest_per_rank"][0] != line["node_digest_per_rank"][1]
    assert not [f for f in os.listdir(tmp_path) if ".tmp" in f]
