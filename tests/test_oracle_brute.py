"""Cross-check the two independent oracles: C set-semantics vs Python brute force over Delta x Delta.

After SPEC.md:557 (acceptance #1: 1,000 random (KB, hypothesis) pairs covering every operator).
"""
import numpy as np

from oracle import brute, setsem
from synth import abox, hyps
from synth.format import COMPILE_COMPAT_PAPER_MAX, flatten


def _run(seed, flags):
    kb = abox.random_tiny_kb(seed)
    shape = abox.kb_shape(kb)
    rng = np.random.default_rng(10_000 + seed)
    trees = [hyps.random_tree(rng, shape, depth=4) for _ in range(8)]
    flat = flatten(trees)
    nodes, kids, roots = flat
    bits, counts = setsem.evaluate(kb, nodes, kids, roots, flags=flags, patterns=flat.patterns)
    res = brute.evaluate(kb, nodes, kids, roots,
                         compat_paper_max=bool(flags & COMPILE_COMPAT_PAPER_MAX), patterns=flat.patterns)
    for i, (h, c) in enumerate(res):
        assert (bits[i] == brute.to_words(h, kb["N"])).all(), (seed, i, trees[i])
        assert tuple(int(v) for v in counts[i]) == c, (seed, i)
    return nodes


def test_random_tiny_vs_brute():
    seen = set()
    for seed in range(130):          # 130 KBs x 8 hypotheses = 1,040 pairs
        nodes = _run(seed, 0)
        seen |= {(int(o), int(f) & 1) for o, f in zip(nodes["op"], nodes["flags"])}
    # every opcode and both role directions were exercised
    assert {o for o, _ in seen} == set(range(14))
    assert {(o, 1) for o in (6, 7, 8, 9, 10)} <= seen


def test_random_tiny_vs_brute_compat():
    for seed in range(500, 540):
        _run(seed, COMPILE_COMPAT_PAPER_MAX)


def test_c1_vs_brute():
    kb = abox.c1_kb()
    trees = hyps.c1_hypotheses(kb)
    nodes, kids, roots = flatten(trees)
    bits, counts = setsem.evaluate(kb, nodes, kids, roots)
    for i, (h, c) in enumerate(brute.evaluate(kb, nodes, kids, roots)):
        assert (bits[i] == brute.to_words(h, 32)).all()
        assert tuple(int(v) for v in counts[i]) == c


def test_threads_do_not_change_results():
    kb = abox.c1_kb()
    nodes, kids, roots = flatten(hyps.c1_hypotheses(kb))
    b1, c1 = setsem.evaluate(kb, nodes, kids, roots, threads=1)
    b4, c4 = setsem.evaluate(kb, nodes, kids, roots, threads=4)
    assert (b1 == b4).all() and (c1 == c4).all()
