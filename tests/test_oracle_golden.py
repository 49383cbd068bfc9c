"""Pin the oracle to hand-worked examples (tests/golden/*.kbt, each citing SPEC.md/PAPER.md)."""
import pytest

from golden_io import all_fixtures, load
from oracle import brute, setsem
from synth.format import COMPILE_COMPAT_PAPER_MAX, flatten


@pytest.mark.parametrize("path", all_fixtures(), ids=lambda p: p.split("/")[-1])
def test_golden_setsem(path):
    kb, cases, flags = load(path)
    flat = flatten([c[1] for c in cases])
    nodes, kids, roots = flat
    bits, counts = setsem.evaluate(kb, nodes, kids, roots, flags=flags, patterns=flat.patterns)
    n = kb["N"]
    for i, (text, _, members, cnt) in enumerate(cases):
        got = {x for x in range(n) if (int(bits[i][x // 32]) >> (x % 32)) & 1}
        assert got == members, text
        if cnt is not None:
            assert tuple(int(v) for v in counts[i]) == cnt, text


@pytest.mark.parametrize("path", all_fixtures(), ids=lambda p: p.split("/")[-1])
def test_golden_brute(path):
    kb, cases, flags = load(path)
    flat = flatten([c[1] for c in cases])
    nodes, kids, roots = flat
    res = brute.evaluate(kb, nodes, kids, roots,
                         compat_paper_max=bool(flags & COMPILE_COMPAT_PAPER_MAX), patterns=flat.patterns)
    for (text, _, members, cnt), (h, c) in zip(cases, res):
        assert h == members, text
        if cnt is not None:
            assert c == cnt, text


def test_empty_contain_rejected():
    """SPEC.md:231 'empty rVal rejected' (reading Q20): the oracle refuses the root."""
    from synth.format import kb_from_sets
    kb = kb_from_sets(2, [[0]], [[]], [], [0], [1], [[(0, b"ab")]])
    flat = flatten([("SCONTAIN", 0, ""), ("SEQUAL", 0, "")])
    with pytest.raises(setsem.OracleError):
        setsem.evaluate(kb, *flat, patterns=flat.patterns)
    with pytest.raises(ValueError):
        brute.evaluate(kb, *flat, patterns=flat.patterns)
    # EQUAL with the empty literal is legal: matches only empty asserted values
    flat = flatten([("SEQUAL", 0, "")])
    bits, _ = setsem.evaluate(kb, *flat, patterns=flat.patterns)
    assert int(bits[0][0]) == 0
