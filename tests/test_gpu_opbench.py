"""NEXT-1 operator micro-benchmarks (tools/opbench.py, the paper's Tables 2 / 4 / card_role / 8)
at the paper's largest size, 10^7 individuals / assertions: every cell's bitset and counts
(and the counts-only variant of the boolean rows) bit-exact against the oracle."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N = 10_000_000


def _opbench():
    import opbench
    return opbench


@pytest.mark.parametrize("op", ["AND", "OR"])
def test_table2_boolean_10m(op):
    ob = _opbench()
    kb = ob.concepts_kb(N, 5, N)
    tree = (op, [("ATOM", i) for i in range(5)])
    for bits in (True, False):
        _, _, ok = ob.measure(kb, tree, 3, True, bits=bits)
        assert ok, (op, bits)


@pytest.mark.parametrize("regime", ["unique", "single"])
def test_table4_card_table8_regimes_10m(regime):
    from synth import abox
    ob = _opbench()
    kb = abox.string_regime_kb(regime, N, seed=N)
    A = ("ATOM", 0)
    cases = [("EXISTS", 0, False, A), ("FORALL", 0, False, A), ("MIN", 3, 0, False, A), ("MAX", 3, 0, False, A),
             ("DRANGE", 0, 1.0, np.inf), ("SEQUAL", 0, b"fixed string value"), ("SCONTAIN", 0, b"string")]
    for tree in cases:
        _, _, ok = ob.measure(kb, tree, 3, True)
        assert ok, (regime, tree[0])
    kb = abox.string_regime_kb(regime, N, seed=N, distinct=True)
    for tree in (("SEQUAL", 0, b"fixed string value0000000007"), ("SCONTAIN", 0, b"value00000007")):
        _, _, ok = ob.measure(kb, tree, 3, True)
        assert ok, (regime, "distinct", tree[0])
