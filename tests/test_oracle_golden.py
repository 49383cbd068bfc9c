"""Pin the oracle to hand-worked examples (tests/golden/*.kbt, each citing SPEC.md/PAPER.md)."""
import pytest

from golden_io import all_fixtures, load
from oracle import brute, setsem
from synth.format import COMPILE_COMPAT_PAPER_MAX, flatten


@pytest.mark.parametrize("path", all_fixtures(), ids=lambda p: p.split("/")[-1])
def test_golden_setsem(path):
    kb, cases, flags = load(path)
    nodes, kids, roots = flatten([c[1] for c in cases])
    bits, counts = setsem.evaluate(kb, nodes, kids, roots, flags=flags)
    n = kb["N"]
    for i, (text, _, members, cnt) in enumerate(cases):
        got = {x for x in range(n) if (int(bits[i][x // 32]) >> (x % 32)) & 1}
        assert got == members, text
        if cnt is not None:
            assert tuple(int(v) for v in counts[i]) == cnt, text


@pytest.mark.parametrize("path", all_fixtures(), ids=lambda p: p.split("/")[-1])
def test_golden_brute(path):
    kb, cases, flags = load(path)
    nodes, kids, roots = flatten([c[1] for c in cases])
    res = brute.evaluate(kb, nodes, kids, roots,
                         compat_paper_max=bool(flags & COMPILE_COMPAT_PAPER_MAX))
    for (text, _, members, cnt), (h, c) in zip(cases, res):
        assert h == members, text
        if cnt is not None:
            assert c == cnt, text
