"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bar (north_star): instance bitsets and TP/FP/FN/TN counts bit-exact (tolerance 0).
"""
import numpy as np
import pytest

from golden_io import all_fixtures, load
from oracle import setsem
from synth import abox, hyps
from synth.format import (COMPILE_COMPAT_PAPER_MAX, COMPILE_NO_CSE, COMPILE_NO_REWRITE, flatten,
                          kb_from_sets)
from test_oracle_identities import (check_compat_table, check_identities, compat_table_kb,
                                    compat_table_trees, degree_closed_forms, identity_kbs,
                                    identity_pairs)

pytestmark = pytest.mark.gpu


def _hedl():
    import paper_2412_00802_b200 as hedl
    hedl.lib()
    return hedl


def gpu_eval(kb, nodes, kids, roots, flags=0, bits=True, eflags=0, ws_limit=None):
    import torch
    hedl = _hedl()
    k = hedl.hedl_kb_load(kb, 0)
    prog = hedl.hedl_compile(k, nodes, kids, roots, flags)
    if ws_limit:
        prog.set_workspace_limit(ws_limit)
    b, c = hedl.hedl_eval_batch(k, prog, 0, len(roots), want_bits=bits, flags=eflags)
    torch.cuda.synchronize()
    return (b.cpu().numpy().view(np.uint32) if bits else None), c, (k, prog)


def assert_parity(kb, trees=None, arrays=None, flags=0, eflags=0, ws_limit=None, tag=""):
    """Bitsets + counts (bitsets requested) and counts alone (the example-projected path) vs the oracle."""
    nodes, kids, roots = arrays if arrays is not None else flatten(trees)
    gb, gc, (k, prog) = gpu_eval(kb, nodes, kids, roots, flags, eflags=eflags, ws_limit=ws_limit)
    ob, oc = setsem.evaluate(kb, nodes, kids, roots, flags=flags, threads=8)
    bad = np.nonzero((gb != ob).any(axis=1) | (gc != oc).any(axis=1))[0] if len(roots) else []
    assert len(bad) == 0, f"{tag}: {len(bad)} mismatching roots, first {bad[:5]}"
    _, gc2 = _hedl().hedl_eval_batch(k, prog, 0, len(roots), want_bits=False, flags=eflags)
    bad = np.nonzero((gc2 != oc).any(axis=1))[0] if len(roots) else []
    assert len(bad) == 0, f"{tag} (counts only): {len(bad)} mismatching roots, first {bad[:5]}"
    return gb, gc


@pytest.mark.parametrize("path", all_fixtures(), ids=lambda p: p.split("/")[-1])
def test_golden_gpu(path):
    kb, cases, flags = load(path)
    nodes, kids, roots = flatten([c[1] for c in cases])
    gb, gc, _ = gpu_eval(kb, nodes, kids, roots, flags)
    n = kb["N"]
    for i, (text, _, members, cnt) in enumerate(cases):
        got = {x for x in range(n) if (int(gb[i][x // 32]) >> (x % 32)) & 1}
        assert got == members, text
        if cnt is not None:
            assert tuple(int(v) for v in gc[i]) == cnt, text


def test_c1_every_constructor():
    kb = abox.c1_kb()
    trees = hyps.c1_hypotheses(kb)
    for fl in (0, COMPILE_NO_CSE, COMPILE_NO_REWRITE | COMPILE_NO_CSE, COMPILE_COMPAT_PAPER_MAX):
        assert_parity(kb, trees, flags=fl, tag=f"C1 flags={fl}")


def test_c1_eval_one_equals_batch():
    hedl = _hedl()
    kb = abox.c1_kb()
    nodes, kids, roots = flatten(hyps.c1_hypotheses(kb))
    gb, gc, (k, prog) = gpu_eval(kb, nodes, kids, roots)
    for i in range(len(roots)):
        b1, c1 = hedl.hedl_eval_one(k, prog, i, want_bits=True)
        assert np.array_equal(b1.cpu().numpy().view(np.uint32), gb[i]) and c1 == tuple(int(v) for v in gc[i])


def test_random_tiny_1000_pairs():
    """SPEC.md:557 acceptance #1 on the GPU: >= 1,000 random (KB, hypothesis) pairs, every operator."""
    for seed in range(130):
        kb = abox.random_tiny_kb(seed)
        rng = np.random.default_rng(10_000 + seed)
        trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=4) for _ in range(8)]
        assert_parity(kb, trees, tag=f"seed {seed}")
        if seed % 13 == 0:
            assert_parity(kb, trees, flags=COMPILE_COMPAT_PAPER_MAX | COMPILE_NO_CSE, tag=f"seed {seed} compat")


def test_tail_masks():
    """SPEC.md:559 acceptance #3 re-expressed for bitsets: N = 0..129 x AND/OR arity {0,1,2,5,32}."""
    for n in list(range(0, 70)) + [95, 96, 97, 127, 128, 129]:
        rng = np.random.default_rng(n)
        concepts = [[i for i in range(n) if rng.random() < 0.5] for _ in range(32)]
        kb = kb_from_sets(n, concepts, [[(i, (i * 7 + 3) % n) for i in range(n)]] if n else [[]], [], [], [])
        trees = []
        for k in (0, 1, 2, 5, 32):
            ops = [("ATOM", j) if j % 3 else ("NOT", ("ATOM", j)) for j in range(k)]
            trees += [("AND", ops), ("OR", ops), ("NOT", ("AND", ops)), ("NOT", ("OR", ops))]
        trees += [("TOP",), ("BOTTOM",), ("FORALL", 0, False, ("BOTTOM",)), ("MAX", 3, 0, True, ("TOP",))]
        gb, _ = assert_parity(kb, trees, flags=COMPILE_NO_REWRITE, tag=f"N={n}")
        if n % 32:
            assert (gb[:, -1] >> np.uint32(n % 32) == 0).all()


@pytest.mark.parametrize("k", range(0, 47, 3))
def test_identities_gpu(k):
    kb = identity_kbs()[k]
    pairs = identity_pairs(abox.kb_shape(kb), 7 * k + 1)
    trees = [t for p in pairs for t in p[:2]]
    gb, _ = assert_parity(kb, trees, flags=COMPILE_NO_REWRITE | COMPILE_NO_CSE, tag=f"identities {k}")
    check_identities(gb, pairs, k)


def test_compat_table_gpu():
    kb = compat_table_kb()
    nodes, kids, roots = flatten(compat_table_trees())
    std, _, _ = gpu_eval(kb, nodes, kids, roots)
    pap, _, _ = gpu_eval(kb, nodes, kids, roots, COMPILE_COMPAT_PAPER_MAX)
    check_compat_table(std, pap)


@pytest.mark.parametrize("kind,E", [("single", 100_000), ("unique", 100_000), ("single", 1_000_000),
                                    ("single", 513), ("single", 4097), ("single", 33)])
def test_regimes(kind, E):
    """PAPER.md:664 single-subject / unique-subject regimes (heavy rows split over CTAs)."""
    kb = abox.regime_kb(kind, E, seed=E)
    T = ("TOP",)
    trees = [("EXISTS", 0, False, ("ATOM", 0)), ("FORALL", 0, False, ("ATOM", 0)),
             ("MIN", E, 0, False, T), ("MIN", E + 1, 0, False, T), ("MAX", E - 1, 0, False, T),
             ("EXACT", E, 0, False, T), ("MIN", E // 3, 0, False, ("ATOM", 1)),
             ("MAX", E // 2, 0, False, ("ATOM", 0)), ("EXISTS", 0, True, ("ATOM", 1)),
             ("DRANGE", 0, 1.0, 1.0), ("DRANGE", 0, 1.5, 2.0)]
    assert_parity(kb, trees, tag=f"{kind} {E}")


def test_determinism_50_reruns():
    """SPEC.md:243 / :558: 50 reruns on a single-subject KB give identical rows and counts."""
    hedl = _hedl()
    import torch
    kb = abox.regime_kb("single", 200_000, seed=1)
    trees = [("MIN", 50_000, 0, False, ("ATOM", 0)), ("EXISTS", 0, False, ("ATOM", 1)),
             ("FORALL", 0, False, ("ATOM", 0)), ("MAX", 100_000, 0, False, ("ATOM", 1))]
    nodes, kids, roots = flatten(trees)
    gb0, gc0, (k, prog) = gpu_eval(kb, nodes, kids, roots)
    for _ in range(50):
        b, c = hedl.hedl_eval_batch(k, prog, 0, len(roots), want_bits=True)
        torch.cuda.synchronize()
        assert np.array_equal(b.cpu().numpy().view(np.uint32), gb0) and np.array_equal(c, gc0)


def test_degree_closed_forms_powerlaw():
    kb = abox.powerlaw_kb(200_000, 4, 2, 8.0, 20_000, 0.7, 1.0, 0.01, 11)
    trees, expect = degree_closed_forms(kb, ks=(1, 2, 8, 33, 513, 5000))
    nodes, kids, roots = flatten(trees)
    gb, _, _ = gpu_eval(kb, nodes, kids, roots)
    for i in range(len(trees)):
        assert np.array_equal(gb[i], expect[i]), trees[i]


def test_powerlaw_random_hypotheses_and_chunking():
    """Power-law KB with heavy rows; random hypotheses; workspace limits forcing many chunks."""
    kb = abox.powerlaw_kb(100_000, 8, 2, 8.0, 5_000, 0.7, 1.2, 0.01, 12, data_round=1)
    rng = np.random.default_rng(12)
    trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=4) for _ in range(300)]
    gb, gc = assert_parity(kb, trees, tag="powerlaw")
    nodes, kids, roots = flatten(trees)
    for lim in (1 << 20, 3 << 20):
        b2, c2, _ = gpu_eval(kb, nodes, kids, roots, ws_limit=lim)
        assert np.array_equal(b2, gb) and np.array_equal(c2, gc)
    b3, c3, _ = gpu_eval(kb, nodes, kids, roots, COMPILE_NO_CSE | COMPILE_NO_REWRITE)
    assert np.array_equal(b3, gb) and np.array_equal(c3, gc)


def test_c2_latency_set():
    kb = abox.c2_kb()
    trees = hyps.c2_hypotheses(kb)
    assert_parity(kb, trees, tag="C2")


def test_refinement_batch_c4_shape_small():
    """C4-style refinement batch on a 200k-individual KB: all counts, all bitsets."""
    kb = abox.powerlaw_kb(200_000, 50, 2, 8.0, 10_000, 0.7, 1.0, 0.01, 4)
    arrays = hyps.batch_arrays("c4", kb, 3000, 4, chunk=1000, workers=1)
    assert_parity(kb, arrays=arrays, tag="c4-small")


def test_errors_gpu():
    hedl = _hedl()
    kb = abox.c1_kb()
    k = hedl.hedl_kb_load(kb, 0)
    for tree, code in [(("DRANGE", 0, float("nan"), 1.0), 4), (("ATOM", 99), 2), (("EXISTS", 7, False, ("TOP",)), 2),
                       (("DRANGE", 3, 0.0, 1.0), 2)]:
        with pytest.raises(hedl.HedlError) as e:
            hedl.hedl_compile(k, *flatten([tree]))
        assert e.value.code == code, tree
    nodes, kids, roots = flatten([("ATOM", 0), ("ATOM", 1)])
    kids = np.array([1], np.uint32)
    nodes["op"][1] = 3          # NOT
    nodes["child_begin"][1] = 0
    nodes["child_count"][1] = 1
    nodes["op"][0] = 3
    nodes["child_count"][0] = 1  # node 0 -> child 1 -> child ... cycle 1 -> 1
    kids = np.array([1, 1], np.uint32)
    nodes["child_begin"][0] = 1
    with pytest.raises(hedl.HedlError) as e:
        hedl.hedl_compile(k, nodes, kids, np.array([0], np.uint32))
    assert e.value.code == 4
    bad = dict(kb)
    bad["neg_ids"] = np.concatenate([kb["neg_ids"], kb["pos_ids"][:1]])
    with pytest.raises(hedl.HedlError) as e:
        hedl.hedl_kb_load(bad, 0)
    assert e.value.code == 3


def test_parallel_compile_equivalent():
    """Sharded compile + lock-free merge (hedl_compile) == single-threaded compile, node for node in count,
    and both equal the oracle; duplicates across shards are merged (global CSE)."""
    import os
    hedl = _hedl()
    kb = abox.powerlaw_kb(30_000, 20, 2, 8.0, 2_000, 0.7, 1.0, 0.02, 31)
    arrays = hyps.batch_arrays("c4", kb, 40_000, 31, chunk=10_000, workers=4)
    nodes, kids, roots = arrays
    k = hedl.hedl_kb_load(kb, 0)
    infos, outs = [], []
    for threads in ("1", "5", "16"):
        os.environ["HEDL_COMPILE_THREADS"] = threads
        try:
            prog = hedl.hedl_compile(k, nodes, kids, roots)
        finally:
            del os.environ["HEDL_COMPILE_THREADS"]
        infos.append(prog.info())
        outs.append(hedl.hedl_eval_batch(k, prog, 0, len(roots))[1])
    assert infos[0]["n_nodes"] == infos[1]["n_nodes"] == infos[2]["n_nodes"]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    sample = np.arange(0, len(roots), 37)
    _, oc = setsem.evaluate(kb, nodes, kids, roots[sample], threads=8, want_bits=False)
    assert np.array_equal(outs[1][sample], oc)


def test_eval_one_latency_path():
    """hedl_eval_one (single-launch interpreter when the sub-DAG fits in shared memory, else the
    batch path) equals the oracle: C2 (all 256), random tiny KBs, a large-N fallback case."""
    hedl = _hedl()
    cases = [(abox.c2_kb(), hyps.c2_hypotheses(abox.c2_kb()))]
    for seed in range(20):
        kb = abox.random_tiny_kb(seed)
        rng = np.random.default_rng(30_000 + seed)
        cases.append((kb, [hyps.random_tree(rng, abox.kb_shape(kb), depth=4) for _ in range(12)]))
    big = abox.powerlaw_kb(3_000_000, 4, 1, 4.0, 600, 0.5, 1.0, 0.001, 8)
    cases.append((big, [("EXISTS", 0, False, ("ATOM", 1)), ("AND", [("ATOM", 0), ("MIN", 2, 0, True, ("ATOM", 2))])]))
    for kb, trees in cases:
        nodes, kids, roots = flatten(trees)
        k = hedl.hedl_kb_load(kb, 0)
        prog = hedl.hedl_compile(k, nodes, kids, roots)
        ob, oc = setsem.evaluate(kb, nodes, kids, roots, threads=8)
        for i in range(len(roots)):
            b1, c1 = hedl.hedl_eval_one(k, prog, i, want_bits=True)
            assert c1 == tuple(int(v) for v in oc[i]), (i, trees[i])
            assert np.array_equal(b1.cpu().numpy().view(np.uint32), ob[i]), (i, trees[i])
            _, c2 = hedl.hedl_eval_one(k, prog, i)
            assert c2 == c1


def test_push_direction_latency_path():
    """Direction-optimising restrictions: on a KB above kPushMinN individuals
    the latency path evaluates a restriction whose counted set S = child ^ cmask holds at most
    N/4 members by walking S through the inverse CSR, else by the pull sweep.  Fillers from
    empty to full density, complemented ones (FORALL counts the complement), every predicate,
    inverse roles, heavy inverse rows (hubs of degree 4,000), nested restrictions: every
    result equals the oracle, bitsets and counts, through hedl_eval_one and a small batch."""
    hedl = _hedl()
    kb = abox.powerlaw_kb(400_000, 12, 2, 8.0, 4000, 0.7, 1.0, 0.01, seed=31)
    A = lambda i: ("ATOM", i)
    trees = []
    for r in range(2):
        for inv in (False, True):
            for c in (A(0), A(5), A(11), ("NOT", A(3)), ("TOP",), ("BOTTOM",), ("AND", [A(1), A(2)])):
                trees += [("EXISTS", r, inv, c), ("FORALL", r, inv, c), ("MIN", 2, r, inv, c), ("MAX", 1, r, inv, c),
                          ("EXACT", 3, r, inv, c), ("MIN", 0, r, inv, c)]
    trees += [("EXISTS", 0, False, ("AND", [A(1), ("FORALL", 1, True, ("OR", [A(2), ("NOT", A(3))]))])),
              ("MIN", 2, 0, True, ("EXISTS", 1, False, A(4))), ("FORALL", 0, False, ("OR", [("EXISTS", 0, False, A(5)),
                                                                                             ("DRANGE", 0, 0.5, np.inf)]))]
    nodes, kids, roots = flatten(trees)
    k = hedl.hedl_kb_load(kb, 0)
    prog = hedl.hedl_compile(k, nodes, kids, roots)
    ob, oc = setsem.evaluate(kb, nodes, kids, roots, threads=8)
    for i in range(len(roots)):
        b1, c1 = hedl.hedl_eval_one(k, prog, i, want_bits=True)
        assert c1 == tuple(int(v) for v in oc[i]), (i, trees[i])
        assert np.array_equal(b1.cpu().numpy().view(np.uint32), ob[i]), (i, trees[i])
    for first in range(0, len(roots), 6):          # groups of <= 8 nodes on the batch path too
        n = min(6, len(roots) - first)
        b, c = hedl.hedl_eval_batch(k, prog, first, n, want_bits=True, flags=2)
        assert np.array_equal(c, oc[first:first + n]) and np.array_equal(b.cpu().numpy().view(np.uint32),
                                                                         ob[first:first + n]), first


def test_free_order_kb_before_program():
    """A program keeps its KB alive: freeing the KB handle first, then the program, leaves the
    library healthy for the next KB (regression: use-after-free on the KB's device id)."""
    hedl = _hedl()
    kb = abox.c1_kb()
    nodes, kids, roots = flatten(hyps.c1_hypotheses(kb))
    for _ in range(3):
        k = hedl.hedl_kb_load(kb, 0)
        prog = hedl.hedl_compile(k, nodes, kids, roots)
        _, c = hedl.hedl_eval_one(k, prog, 3)
        k.free()                        # program still alive: evaluation must keep working
        _, c2 = hedl.hedl_eval_batch(k, prog, 3, 1)
        assert tuple(int(v) for v in c2[0]) == c
        prog.free()


def test_drange_groups_long_segments():
    """Range groups (several nodes on one data property in one launch: k_drange_multi) over
    value segments of 0..12 values (the kernel caches four per individual and binary-searches
    longer segments), NaN-free sorted per individual, with bounds at, between and outside the
    values, empty and inverted ranges, +-inf; 1, 2, 31, 32, 33 and 70 nodes per group; full
    rows (bits requested) and the example-projected counts path."""
    rng = np.random.default_rng(77)
    kb = abox.powerlaw_kb(9000 + 5, 6, 1, 4.0, 300, 0.0, 1.0, 0.05, seed=12)
    N = kb["N"]
    cnt = rng.integers(0, 13, size=N)
    cnt[rng.random(N) < 0.3] = 0
    subj = np.repeat(np.arange(N, dtype=np.uint32), cnt)
    vals = np.round(rng.normal(0, 2, size=len(subj)), 1).astype(np.float32)
    kb["data_off"] = np.array([0, len(subj)], np.uint64)
    kb["data_subj"], kb["data_val"] = subj, vals
    bounds = [-np.inf, -3.0, -1.0, -0.5, 0.0, 0.1, 0.5, 1.0, 2.5, 4.0, np.inf]
    ranges = [(lo, hi) for lo in bounds for hi in bounds]          # incl. lo > hi (empty)
    for k in (1, 2, 31, 32, 33, 70):
        trees = [("DRANGE", 0, float(lo), float(hi)) for lo, hi in ranges[:k]]
        trees += [("AND", [("ATOM", q % 6), ("DRANGE", 0, float(lo), float(hi))]) for q, (lo, hi) in enumerate(ranges[:k])]
        trees += [("EXISTS", 0, q % 2 == 1, ("DRANGE", 0, float(lo), float(hi))) for q, (lo, hi) in enumerate(ranges[:k])]
        assert_parity(kb, trees, tag=f"drange groups k={k}")
