"""Generators are seeded and deterministic; the s-expression reader round-trips."""
import numpy as np

from synth import abox, hyps
from synth.format import flatten, parse, tree_to_text


def test_generators_deterministic():
    a, b = abox.c1_kb(), abox.c1_kb()
    for k in a:
        assert np.asarray(a[k]).tobytes() == np.asarray(b[k]).tobytes()
    k1 = abox.powerlaw_kb(2000, 3, 2, 8.0, 300, 0.7, 1.2, 0.01, 9)
    k2 = abox.powerlaw_kb(2000, 3, 2, 8.0, 300, 0.7, 1.2, 0.01, 9)
    for k in k1:
        assert np.asarray(k1[k]).tobytes() == np.asarray(k2[k]).tobytes()
    # forced heavy row and tail bits zero
    assert (k1["edge_subj"][: k1["role_edge_off"][1]] == 0).sum() == 300
    n = k1["N"]
    if n % 32:
        assert (k1["concept_bits"][:, -1] >> np.uint32(n % 32) == 0).all()


def test_parse_roundtrip():
    names = {"concepts": ["A", "B"], "roles": ["r", "s"], "data": ["d"]}
    for text in ["(AND A (NOT B))", "(SOME (INV r) (OR A B))", "(ONLY s TOP)", "(MIN 2 r A)",
                 "(MAX 0 (INV s) BOTTOM)", "(EXACTLY 3 r (NOT (AND)))", "(DRANGE d -inf 0.5)"]:
        t = parse(text, names)
        assert parse(tree_to_text(t, names), names) == t
    assert parse("(SOME (INV (INV r)) A)", names) == parse("(SOME r A)", names)


def test_c1_covers_every_opcode():
    kb = abox.c1_kb()
    nodes, _, roots = flatten(hyps.c1_hypotheses(kb))
    assert len(roots) == 64
    assert set(nodes["op"].tolist()) == set(range(12))
    assert {(int(o), int(f)) for o, f in zip(nodes["op"], nodes["flags"]) if o in (6, 7, 8, 9, 10)} >= \
        {(o, f) for o in (6, 7, 8, 9) for f in (0, 1)}


def test_batch_arrays_concat_consistent():
    kb = abox.powerlaw_kb(5000, 10, 2, 8.0, 200, 0.7, 1.0, 0.01, 4)
    nodes, kids, roots = hyps.batch_arrays("c4", kb, 3000, 4, chunk=1000, workers=1)
    assert len(roots) == 3000
    assert (roots < len(nodes)).all() and (kids < len(nodes)).all()
    assert (nodes["child_begin"].astype(np.int64) + nodes["child_count"] <= len(kids)).all()
