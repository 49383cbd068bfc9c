"""Device-side compile (hedl_compile_device) vs the oracle,
element by element (bitsets + counts, bit-exact), and vs the host compiler's program shape."""
import numpy as np
import pytest

from golden_io import all_fixtures, load
from oracle import setsem
from synth import abox, hyps
from synth.format import COMPILE_COMPAT_PAPER_MAX, COMPILE_NO_CSE, COMPILE_NO_REWRITE, flatten
from test_gpu_parity import _hedl

pytestmark = pytest.mark.gpu


def dev_parity(kb, nodes, kids, roots, flags=0, eflags=0, tag=""):
    import torch
    hedl = _hedl()
    k = hedl.hedl_kb_load(kb, 0)
    prog = hedl.hedl_compile_device(k, nodes, kids, roots, flags)
    b, c = hedl.hedl_eval_batch(k, prog, 0, len(roots), want_bits=True, flags=eflags)
    torch.cuda.synchronize()
    gb = b.cpu().numpy().view(np.uint32)
    ob, oc = setsem.evaluate(kb, nodes, kids, roots, flags=flags, threads=8)
    bad = np.nonzero((gb != ob).any(axis=1) | (c != oc).any(axis=1))[0] if len(roots) else []
    assert len(bad) == 0, f"{tag}: {len(bad)} mismatching roots, first {bad[:5]}"
    _, c2 = hedl.hedl_eval_batch(k, prog, 0, len(roots), want_bits=False, flags=eflags)
    bad = np.nonzero((c2 != oc).any(axis=1))[0] if len(roots) else []
    assert len(bad) == 0, f"{tag} (counts only): {len(bad)} mismatching roots"
    return k, prog


@pytest.mark.parametrize("path", [p for p in all_fixtures() if not p.endswith("strings.kbt")],
                         ids=lambda p: p.split("/")[-1])
def test_golden_device_compile(path):
    kb, cases, flags = load(path)
    nodes, kids, roots = flatten([c[1] for c in cases])
    dev_parity(kb, nodes, kids, roots, flags, tag=path)


def test_c1_flags_device_compile():
    kb = abox.c1_kb()
    nodes, kids, roots = flatten(hyps.c1_hypotheses(kb))
    for fl in (0, COMPILE_NO_CSE, COMPILE_NO_REWRITE | COMPILE_NO_CSE, COMPILE_NO_REWRITE, COMPILE_COMPAT_PAPER_MAX):
        dev_parity(kb, nodes, kids, roots, fl, tag=f"C1 flags={fl}")


def test_random_tiny_device_compile():
    for seed in range(80):
        kb = abox.random_tiny_kb(seed, n_strings=0)
        rng = np.random.default_rng(seed + 77)
        trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=4) for _ in range(12)]
        f = flatten(trees)
        dev_parity(kb, *f, tag=f"tiny {seed}")
        fs = flatten(trees, share=True)                       # shared subtrees (a DAG input)
        dev_parity(kb, *fs, tag=f"tiny shared {seed}")


def test_refinement_batch_device_compile():
    """C4-shaped refinement batch (20k hypotheses, 300k individuals) incl. lane-packed paths;
    the device program has the host program's node counts up to root-only duplicates."""
    hedl = _hedl()
    kb = abox.powerlaw_kb(300_000, 20, 2, 8.0, 3000, data_frac=0.7, data_vals_mean=1.0, ex_frac=0.01, seed=9)
    nodes, kids, roots = hyps.batch_arrays("c4", kb, 20_000, seed=3)
    k, prog = dev_parity(kb, nodes, kids, roots, tag="refine")
    dev_parity(kb, nodes, kids, roots, eflags=2, tag="refine per-node")
    host = hedl.hedl_compile(k, nodes, kids, roots)
    hi, di = host.info(), prog.info()
    assert di["n_restrict"] == hi["n_restrict"] and di["n_drange"] == hi["n_drange"]
    assert di["n_levels"] == hi["n_levels"]
    assert abs(di["n_nodes"] - hi["n_nodes"]) <= hi["n_nodes"] // 10


def test_device_compile_errors():
    hedl = _hedl()
    kb = abox.c1_kb()
    k = hedl.hedl_kb_load(kb, 0)
    bad_cases = [
        ([("ATOM", 99)], 2),
        ([("EXISTS", 5, False, ("TOP",))], 2),
        ([("DRANGE", 0, float("nan"), 1.0)], 4),
        ([("SEQUAL", 0, b"x")], 8),
    ]
    for trees, code in bad_cases:
        f = flatten(trees)
        with pytest.raises(hedl.HedlError) as e:
            hedl.hedl_compile_device(k, *f)
        assert e.value.code == code, trees
    nodes, kids, roots = flatten([("AND", [("ATOM", 0), ("ATOM", 1)])])
    kids2 = kids.copy()
    kids2[0] = 2                                           # a child after its parent
    with pytest.raises(hedl.HedlError) as e:
        hedl.hedl_compile_device(k, nodes, kids2, roots)
    assert e.value.code == 4
    with pytest.raises(hedl.HedlError) as e:
        hedl.hedl_compile_device(k, nodes, kids, np.array([7], np.uint32))
    assert e.value.code == 2
    # an invalid node nobody reaches is not an error (as for the host compiler)
    nodes2 = np.concatenate([nodes, flatten([("ATOM", 99)])[0]])
    prog = hedl.hedl_compile_device(k, nodes2, kids, roots)
    assert prog.info()["n_roots"] == 1


def test_device_plan_subranges_and_fallback():
    """Device plans for sub-ranges of the roots, eval_one above the interpreter's size, and the
    host-planner fallback when the batch needs several chunks (tiny workspace limit)."""
    import torch
    hedl = _hedl()
    kb = abox.powerlaw_kb(120_000, 12, 2, 6.0, 2000, data_frac=0.5, data_vals_mean=1.2, ex_frac=0.02, seed=5)
    nodes, kids, roots = hyps.batch_arrays("c4", kb, 3000, seed=8)
    ob, oc = setsem.evaluate(kb, nodes, kids, roots, threads=8)
    k = hedl.hedl_kb_load(kb, 0)
    prog = hedl.hedl_compile_device(k, nodes, kids, roots)
    for a, b in ((0, 1), (5, 700), (2999, 3000), (100, 3000)):
        bits, c = hedl.hedl_eval_batch(k, prog, a, b - a, want_bits=True)
        assert np.array_equal(bits.cpu().numpy().view(np.uint32), ob[a:b]) and np.array_equal(c, oc[a:b]), (a, b)
        _, c = hedl.hedl_eval_batch(k, prog, a, b - a, want_bits=False)
        assert np.array_equal(c, oc[a:b]), (a, b)
    for i in (0, 17, 2999):
        b1, c1 = hedl.hedl_eval_one(k, prog, i, want_bits=True)
        assert np.array_equal(b1.cpu().numpy().view(np.uint32), ob[i]) and c1 == tuple(int(v) for v in oc[i])
    p2 = hedl.hedl_compile_device(k, nodes, kids, roots)
    p2.set_workspace_limit(1 << 20)                      # 1 MiB: many chunks -> host planner
    bits, c = hedl.hedl_eval_batch(k, p2, 0, 3000, want_bits=True)
    torch.cuda.synchronize()
    assert np.array_equal(bits.cpu().numpy().view(np.uint32), ob) and np.array_equal(c, oc)


def test_device_compile_deep_and_shared_dags():
    """Levels on the device: one bounded depth-first pass (k_dc_level_dfs), falling back to
    relaxation passes when a sub-DAG is deeper than the walk's stack (a 30-deep chain of
    restrictions) or too shared for its visit budget (a ladder DAG whose paths double per
    step, emitted with shared subtrees) -- both vs the oracle, next to plain trees."""
    kb = abox.powerlaw_kb(3000, 8, 2, 5.0, 200, 0.5, 1.0, 0.05, seed=9)
    A = lambda i: ("ATOM", i)
    chain = A(0)
    for d in range(30):
        chain = ("EXISTS", d % 2, d % 3 == 0, chain) if d % 4 else ("AND", [chain, ("NOT", A(d % 8))])
    def ladder(steps):
        t = A(1)
        for d in range(steps):
            t = ("AND", [t, ("OR", [t, A((d + 2) % 8)])]) if d % 2 else ("OR", [t, ("EXISTS", 0, False, t)])
        return t
    for share, steps in ((False, 10), (True, 20)):       # unshared: 2^steps paths as a tree
        lad = ladder(steps)
        trees = [chain, lad, ("EXISTS", 1, True, lad), A(3), ("FORALL", 0, False, A(2))]
        nodes, kids, roots = flatten(trees, share=share)
        dev_parity(kb, nodes, kids, roots, tag=f"deep/shared DAGs share={share}")
