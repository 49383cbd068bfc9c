"""Pin the C oracle with DL identities, closed forms and invariants (SURVEY 8(c) "What pins each part").

Each identity is checked on seeded random KBs, evaluating both sides as
separate hypotheses (no rewriting), so a dropped term, wrong sign, wrong
index or transposed operand in any operator fails at least one of them.
"""
import numpy as np
import pytest

from oracle import setsem
from synth import abox, hyps
from synth.format import COMPILE_COMPAT_PAPER_MAX, flatten, kb_from_sets

T, B = ("TOP",), ("BOTTOM",)


def NOT(x): return ("NOT", x)
def AND(*x): return ("AND", list(x))
def OR(*x): return ("OR", list(x))
def EX(r, inv, c): return ("EXISTS", r, inv, c)
def ALL(r, inv, c): return ("FORALL", r, inv, c)
def MIN(n, r, inv, c): return ("MIN", n, r, inv, c)
def MAX(n, r, inv, c): return ("MAX", n, r, inv, c)
def EQ(n, r, inv, c): return ("EXACT", n, r, inv, c)


def identity_pairs(shape, seed, k=6):
    """(lhs, rhs, relation) with relation 'eq' or 'sub' (lhs subset of rhs).  Shared with GPU tests."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(k):
        C = hyps.random_tree(rng, shape, depth=3)
        D = hyps.random_tree(rng, shape, depth=3)
        out += [(NOT(NOT(C)), C, "eq"),
                (NOT(AND(C, D)), OR(NOT(C), NOT(D)), "eq"),
                (NOT(OR(C, D)), AND(NOT(C), NOT(D)), "eq"),
                (AND(C, NOT(C)), B, "eq"), (OR(C, NOT(C)), T, "eq"),
                (AND(C, D), AND(D, C), "eq"), (AND(C, C), C, "eq"), (OR(C, C), C, "eq"),
                (AND(C, D), C, "sub"), (C, OR(C, D), "sub")]
        if shape["R"]:
            r, inv = int(rng.integers(shape["R"])), bool(rng.integers(2))
            n = int(rng.integers(0, 5))
            out += [(EX(r, inv, C), MIN(1, r, inv, C), "eq"),                 # exists = >=1
                    (ALL(r, inv, C), NOT(EX(r, inv, NOT(C))), "eq"),          # forall = not exists not
                    (MAX(n, r, inv, C), NOT(MIN(n + 1, r, inv, C)), "eq"),    # <=n = not >=(n+1)
                    (EQ(n, r, inv, C), AND(MIN(n, r, inv, C), MAX(n, r, inv, C)), "eq"),
                    (MIN(0, r, inv, C), T, "eq"),
                    (MIN(n + 1, r, inv, C), MIN(n, r, inv, C), "sub"),       # chain
                    (EX(r, inv, B), B, "eq"), (ALL(r, inv, T), T, "eq"),
                    (EX(r, inv, C), EX(r, inv, OR(C, D)), "sub"),            # monotone
                    (C, ALL(r, not inv, EX(r, inv, C)), "sub"),              # ALCI tautology
                    (EX(r, inv, OR(C, D)), OR(EX(r, inv, C), EX(r, inv, D)), "eq"),
                    (ALL(r, inv, AND(C, D)), AND(ALL(r, inv, C), ALL(r, inv, D)), "eq")]
        if shape.get("S"):
            s_, v = int(rng.integers(shape["S"])), hyps.STR_PATTERNS[int(rng.integers(len(hyps.STR_PATTERNS)))]
            out += [(("SEQUAL", s_, v), ("SCONTAIN", s_, v), "sub"),           # equality is a containment
                    (("SCONTAIN", s_, v), ("SCONTAIN", s_, v[:1]), "sub"),     # shorter substring
                    (("SCONTAIN", s_, v + "\x00never"), B, "eq")]              # no asserted value holds NUL
    return out


def identity_kbs():
    out = [abox.random_tiny_kb(s) for s in range(40)]
    out += [abox.random_tiny_kb(s, n=300, n_concepts=3, n_roles=2, n_data=1, n_strings=1) for s in range(100, 106)]
    out.append(abox.c1_kb())
    return out


def bits_to_int(row):
    return int.from_bytes(np.asarray(row, dtype="<u4").tobytes(), "little")


def check_identities(bits, pairs, tag):
    for i, (l, r, rel) in enumerate(pairs):
        a, b = bits_to_int(bits[2 * i]), bits_to_int(bits[2 * i + 1])
        if rel == "eq":
            assert a == b, (tag, l, r)
        else:
            assert a & ~b == 0, (tag, l, r)


@pytest.mark.parametrize("k", range(47))
def test_identities(k):
    kb = identity_kbs()[k]
    pairs = identity_pairs(abox.kb_shape(kb), 7 * k + 1)
    trees = [t for p in pairs for t in p[:2]]
    nodes, kids, roots = flatten(trees)
    bits, _ = setsem.evaluate(kb, nodes, kids, roots)
    check_identities(bits, pairs, k)


def _edges(kb, r):
    off = kb["role_edge_off"]
    return (kb["edge_subj"][off[r]:off[r + 1]].astype(np.int64),
            kb["edge_obj"][off[r]:off[r + 1]].astype(np.int64))


def set_bits(n, ids):
    w = np.zeros((n + 31) // 32, dtype=np.uint32)
    ids = np.unique(np.asarray(ids, dtype=np.int64))
    np.bitwise_or.at(w, ids // 32, (np.uint32(1) << (ids % 32).astype(np.uint32)))
    return w


def degree_closed_forms(kb, roles=(0, 1), ks=(1, 2, 3, 7)):
    """exists r.TOP = {x: has a successor}; exists r^-.TOP = range of r;
    >=k r.TOP = {x : #distinct successors >= k} (numpy unique/bincount).  -> (trees, expected rows)."""
    n = kb["N"]
    trees, expect = [], []
    for r in roles:
        s, o = _edges(kb, r)
        key = np.unique(s * n + o)
        us, uo = key // n, key % n
        trees += [EX(r, False, T), EX(r, True, T)]
        expect += [set_bits(n, us), set_bits(n, uo)]
        deg = np.bincount(us, minlength=n)
        ideg = np.bincount(uo, minlength=n)
        for k in ks:
            trees.append(MIN(k, r, False, T))
            expect.append(set_bits(n, np.nonzero(deg >= k)[0]))
            trees.append(MIN(k, r, True, T))
            expect.append(set_bits(n, np.nonzero(ideg >= k)[0]))
    return trees, expect


@pytest.mark.parametrize("seed", range(12))
def test_closed_forms_degree(seed):
    kb = abox.random_tiny_kb(seed, n=200 + seed, n_roles=2) if seed % 2 else \
        abox.powerlaw_kb(3000, 3, 2, 6.0, 400, 0.5, 1.0, 0.05, seed)
    trees, expect = degree_closed_forms(kb)
    nodes, kids, roots = flatten(trees)
    bits, _ = setsem.evaluate(kb, nodes, kids, roots)
    for i in range(len(trees)):
        assert (bits[i] == expect[i]).all(), (seed, trees[i])


def test_single_subject_hub_threshold():
    """PAPER.md:664 'Single subject' regime: one hub of degree E; >=E holds, >=E+1 fails."""
    for E in (1, 31, 32, 33, 1000, 5000):
        kb = abox.regime_kb("single", E, seed=E)
        trees = [MIN(E, 0, False, T), MIN(E + 1, 0, False, T), MAX(E - 1, 0, False, T),
                 EQ(E, 0, False, T), EX(0, True, T)]
        nodes, kids, roots = flatten(trees)
        bits, _ = setsem.evaluate(kb, nodes, kids, roots)
        hub = set_bits(kb["N"], [0])
        assert (bits[0] == hub).all() and not bits[1].any()
        assert (bits[2] == (~hub & set_bits(kb["N"], range(kb["N"])))).all()
        assert (bits[3] == hub).all()
        assert (bits[4] == set_bits(kb["N"], range(1, E + 1))).all()


def test_inverse_is_swap():
    """(r^-)^- = r: exists r^-.C on a KB whose role lists are swapped equals exists r.C."""
    for seed in range(10):
        kb = abox.random_tiny_kb(seed, n=50, n_roles=1)
        sw = dict(kb)
        sw["edge_subj"], sw["edge_obj"] = kb["edge_obj"], kb["edge_subj"]
        shape = dict(abox.kb_shape(kb), R=0)      # the filler must not itself use the role
        rng = np.random.default_rng(seed)
        C = hyps.random_tree(rng, shape, depth=3)
        for mk in (lambda inv: EX(0, inv, C), lambda inv: ALL(0, inv, C),
                   lambda inv: MIN(2, 0, inv, C), lambda inv: MAX(1, 0, inv, C)):
            a, _ = setsem.evaluate(kb, *flatten([mk(False)]))
            b, _ = setsem.evaluate(sw, *flatten([mk(True)]))
            assert (a == b).all()


def test_duplicates_collapse():
    """Role extensions are sets: duplicating every assertion changes nothing."""
    for seed in range(10):
        kb = abox.random_tiny_kb(seed, n=30)
        dup = dict(kb)
        dup["edge_subj"] = np.repeat(kb["edge_subj"], 2)
        dup["edge_obj"] = np.repeat(kb["edge_obj"], 2)
        dup["role_edge_off"] = kb["role_edge_off"] * 2
        shape = abox.kb_shape(kb)
        rng = np.random.default_rng(seed)
        trees = [hyps.random_tree(rng, shape, depth=3) for _ in range(10)]
        nodes, kids, roots = flatten(trees)
        a, ca = setsem.evaluate(kb, nodes, kids, roots)
        b, cb = setsem.evaluate(dup, nodes, kids, roots)
        assert (a == b).all() and (ca == cb).all()


def range_reference(kb, d, lo, hi):
    """exists d.[lo,hi] via a global (value, subject) sort + two binary searches + scatter."""
    a0, a1 = int(kb["data_off"][d]), int(kb["data_off"][d + 1])
    v = kb["data_val"][a0:a1].astype(np.float32)
    s = kb["data_subj"][a0:a1].astype(np.int64)
    order = np.argsort(v, kind="stable")                 # NaN sorts last
    vs, ss = v[order], s[order]
    a = np.searchsorted(vs, np.float32(lo), side="left")
    b = np.searchsorted(vs, np.float32(hi), side="right")
    return set_bits(kb["N"], ss[a:max(a, b)])


def test_numeric_range_independent_algorithm():
    pool = np.array([-np.inf, -2.0, -1.5, -0.0, 0.0, 0.5, 1.0, 2.25, 3.0, np.inf], np.float32)
    for seed in range(15):
        kb = abox.random_tiny_kb(seed, n=60, n_data=1) if seed < 10 else \
            abox.powerlaw_kb(5000, 1, 1, 2.0, 50, 0.7, 1.5, 0.01, seed, data_round=1)
        n = kb["N"]
        rng = np.random.default_rng(seed)
        trees, expect = [], []
        for _ in range(30):
            lo, hi = (rng.choice(pool), rng.choice(pool)) if seed < 10 else \
                tuple(np.float32(x) for x in np.round(rng.normal(0, 1, 2), 1))
            trees.append(("DRANGE", 0, float(lo), float(hi)))
            expect.append(range_reference(kb, 0, lo, hi))
        nodes, kids, roots = flatten(trees)
        bits, _ = setsem.evaluate(kb, nodes, kids, roots)
        for i in range(len(trees)):
            assert (bits[i] == expect[i]).all(), (seed, trees[i])
        # [-inf,+inf] = individuals with >= 1 non-NaN value; [v,+inf] u [-inf,v] = the same set
        v, s = kb["data_val"], kb["data_subj"]
        nodes, kids, roots = flatten([("DRANGE", 0, -np.inf, np.inf),
                                      OR(("DRANGE", 0, 0.5, np.inf), ("DRANGE", 0, -np.inf, 0.5))])
        bits, _ = setsem.evaluate(kb, nodes, kids, roots)
        assert (bits[0] == set_bits(n, s[~np.isnan(v)])).all() and (bits[0] == bits[1]).all()


def test_constant_value_regime():
    """every value fixed to one constant -> all-or-nothing."""
    kb = abox.regime_kb("unique", 1000, seed=3)
    subj = set_bits(kb["N"], kb["data_subj"])
    trees = [("DRANGE", 0, 1.0, 1.0), ("DRANGE", 0, 1.0000001, np.inf), ("DRANGE", 0, -np.inf, 1.0)]
    bits, _ = setsem.evaluate(kb, *flatten(trees))
    assert (bits[0] == subj).all() and not bits[1].any() and (bits[2] == subj).all()


def test_coverage_invariants():
    for seed in range(20):
        kb = abox.random_tiny_kb(seed, n=64)
        shape = abox.kb_shape(kb)
        rng = np.random.default_rng(seed)
        C = [hyps.random_tree(rng, shape, depth=3) for _ in range(5)]
        trees = [T, B] + C + [NOT(c) for c in C]
        bits, cnt = setsem.evaluate(kb, *flatten(trees))
        P, N = len(kb["pos_ids"]), len(kb["neg_ids"])
        assert tuple(cnt[0]) == (P, N, 0, 0) and tuple(cnt[1]) == (0, 0, P, N)
        assert (cnt[:, 0] + cnt[:, 2] == P).all() and (cnt[:, 1] + cnt[:, 3] == N).all()
        for i in range(5):
            assert cnt[2 + i, 0] + cnt[7 + i, 0] == P and cnt[2 + i, 1] + cnt[7 + i, 1] == N
        # library popcount of the returned rows against the example masks
        pw, nw = set_bits(64, kb["pos_ids"]), set_bits(64, kb["neg_ids"])
        assert (np.bitwise_count(bits & pw).sum(1) == cnt[:, 0]).all()
        assert (np.bitwise_count(bits & nw).sum(1) == cnt[:, 1]).all()


def compat_table_kb():
    """Individual c (0..10) has exactly c successors, all in concept F."""
    n = 11 + 55
    pairs, nxt = [], 11
    for c in range(11):
        for _ in range(c):
            pairs.append((c, nxt))
            nxt += 1
    return kb_from_sets(n, [list(range(11, n))], [pairs], [], [], [])


def compat_table_trees():
    trees = []
    for rv in range(11):
        trees += [MIN(rv, 0, False, ("ATOM", 0)), EQ(rv, 0, False, ("ATOM", 0)),
                  MAX(rv, 0, False, ("ATOM", 0))]
    return trees


def check_compat_table(std, pap):
    bit = lambda row, i: (int(row[i // 32]) >> (i % 32)) & 1
    for rv in range(11):
        for c in range(11):
            assert bit(std[3 * rv], c) == (c >= rv)
            assert bit(std[3 * rv + 1], c) == (c == rv)
            assert bit(std[3 * rv + 2], c) == (c <= rv)
            assert bit(pap[3 * rv + 2], c) == (0 < c <= rv)
            assert bit(pap[3 * rv], c) == (c >= rv)


def test_compat_max_exhaustive_table():
    """SPEC.md:565 acceptance #9: counters 0..10 x rVal 0..10 for MIN / EXACTLY / MAX,
    MAX both standard (Q2) and the paper's cVal>0 guard."""
    kb = compat_table_kb()
    nodes, kids, roots = flatten(compat_table_trees())
    std, _ = setsem.evaluate(kb, nodes, kids, roots)
    pap, _ = setsem.evaluate(kb, nodes, kids, roots, flags=COMPILE_COMPAT_PAPER_MAX)
    check_compat_table(std, pap)


def test_errors():
    kb = abox.c1_kb()
    with pytest.raises(setsem.OracleError) as e:
        setsem.evaluate(kb, *flatten([("DRANGE", 0, float("nan"), 1.0)]))
    assert e.value.code == 4
    with pytest.raises(setsem.OracleError) as e:
        setsem.evaluate(kb, *flatten([("ATOM", 99)]))
    assert e.value.code == 2
    bad = dict(kb)
    bad["neg_ids"] = np.concatenate([kb["neg_ids"], kb["pos_ids"][:1]])
    with pytest.raises(setsem.OracleError) as e:
        setsem.OracleKB(bad)
    assert e.value.code == 3
