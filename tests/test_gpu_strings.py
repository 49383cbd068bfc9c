"""GPU parity of the string concrete-role restrictions (Algs. 11-14,
PAPER.md:400-517) against the oracle, element by element (bit-exact: integer/byte work)."""
import numpy as np
import pytest

from oracle import setsem
from synth import abox, hyps
from synth.format import flatten, kb_from_sets
from test_gpu_parity import _hedl, assert_parity, gpu_eval

pytestmark = pytest.mark.gpu


def test_string_kb_medium_parity():
    """N = 70,000 (several tiles, ragged tail, above the latency interpreter's limit), two string
    roles, Zipf-shared values, hub subjects with 150-300 distinct values (warp-scanned rows),
    embedded NUL bytes, duplicate assertions."""
    kb = abox.string_kb(70_001, seed=1)
    trees = hyps.string_hypotheses(kb, 300, seed=3)
    assert_parity(kb, trees, tag="string_kb")
    assert_parity(kb, trees, eflags=2, tag="string_kb per-node")


def test_string_hub_rows():
    """Long rows: a subject with 5,000 distinct values; the match sits first, last, or nowhere."""
    n = 3000
    vals = [b"v%05d" % i for i in range(5000)]
    strings = [[(7, v) for v in vals] + [(8, vals[-1]), (9, b"x")]]
    kb = kb_from_sets(n, [list(range(0, n, 2))], [[]], [], [7, 8], [9, 10], strings)
    trees = [("SCONTAIN", 0, b"v00000"), ("SCONTAIN", 0, b"v04999"), ("SCONTAIN", 0, b"nope"),
             ("SEQUAL", 0, b"v02500"), ("SCONTAIN", 0, b"0"), ("SEQUAL", 0, b"x"), ("SCONTAIN", 0, b"9")]
    gb, gc = assert_parity(kb, trees, tag="hub")
    assert gb[2].sum() == 0


@pytest.mark.parametrize("kind", ["single", "unique"])
@pytest.mark.parametrize("E", [10, 100_000, 1_000_000])
def test_string_regimes(kind, E):
    """Table 8's string rows: single / unique subject, every value one constant."""
    kb = abox.string_regime_kb(kind, E, seed=E)
    trees = [("SEQUAL", 0, b"fixed string value"), ("SEQUAL", 0, b"other"), ("SCONTAIN", 0, b"string"),
             ("SCONTAIN", 0, b"strinG"), ("SCONTAIN", 0, b"fixed string value!"),
             ("AND", [("ATOM", 0), ("SCONTAIN", 0, b"d s")])]
    assert_parity(kb, trees, tag=f"{kind} {E}")


def test_equal_short_circuit_and_contain_dedupe():
    """An EQUAL literal no assertion holds compiles to BOTTOM with no string node;
    equal CONTAIN patterns share one node."""
    hedl = _hedl()
    kb = kb_from_sets(40, [[1, 2]], [[]], [], [1], [2], [[(1, b"abc"), (2, b"abd")]])
    k = hedl.hedl_kb_load(kb, 0)
    f = flatten([("SEQUAL", 0, b"zzz"), ("SEQUAL", 0, b"abc"), ("SCONTAIN", 0, b"ab"),
                 ("OR", [("SCONTAIN", 0, b"ab"), ("ATOM", 0)])])
    prog = hedl.hedl_compile(k, *f)
    assert prog.info()["n_string"] == 2
    b, c = hedl.hedl_eval_batch(k, prog, 0, 4, want_bits=True)
    b = b.cpu().numpy().view(np.uint32)
    assert b[0].sum() == 0 and int(b[1][0]) == 2 and int(b[2][0]) == 6
    for i in range(4):
        b1, c1 = hedl.hedl_eval_one(k, prog, i, want_bits=True)
        assert np.array_equal(b1.cpu().numpy().view(np.uint32), b[i]) and c1 == tuple(int(v) for v in c[i])


def test_string_errors():
    hedl = _hedl()
    kb = kb_from_sets(4, [[0]], [[]], [], [0], [1], [[(0, b"a")]])
    k = hedl.hedl_kb_load(kb, 0)
    for tree, code in ((("SCONTAIN", 0, b""), 4), (("SEQUAL", 1, b"a"), 2)):
        with pytest.raises(hedl.HedlError) as e:
            hedl.hedl_compile(k, *flatten([tree]))
        assert e.value.code == code
    nodes, kids, roots = flatten([("SEQUAL", 0, b"a")])
    with pytest.raises(hedl.HedlError) as e:                  # pattern id beyond the table
        hedl.hedl_compile_ex(k, nodes, kids, roots, 0, [])
    assert e.value.code == 2
    # EQUAL with the empty literal is legal (matches assertions whose value is empty)
    kb2 = kb_from_sets(4, [[0]], [[]], [], [0], [1], [[(0, b""), (2, b"q")]])
    assert_parity(kb2, [("SEQUAL", 0, b""), ("SCONTAIN", 0, b"q")], tag="empty equal")


def test_random_tiny_strings():
    """Random tiny KBs with string roles x random trees mixing every constructor."""
    for seed in range(60):
        kb = abox.random_tiny_kb(seed, n_strings=2)
        rng = np.random.default_rng(seed)
        trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=4) for _ in range(12)]
        assert_parity(kb, trees, tag=f"tiny {seed}")
