"""Seeded hypothesis generators (trees; flatten with synth.format.flatten).

The paper defines no refinement operator (the learner is out of scope,
SURVEY 8(d)); the refinement-style generator below follows SURVEY 8(d)'s
recipe: a seeded beam from TOP where each child is its parent plus one
downward step, siblings emitted contiguously so they share subtrees.
"""
from __future__ import annotations

import math
from typing import List, Optional

import numpy as np

INF = float("inf")


# ------------------------------------------------------------------------------
# random trees (cover every constructor)


STR_PATTERNS = ["Smith", "Alice Smith", "Bob", "b", "carbon", "c", "CARBON", "bond", "missing", "Ab", "a",
                "\u00e9", '"', "tab\t", "Smithers", "xyz"]


def random_tree(rng, shape: dict, depth: int = 4, n_max: int = 4, allow_drange=True):
    C, R, D = shape["C"], shape["R"], shape["D"]
    S = shape.get("S", 0)
    leaf_kinds = ["TOP", "BOTTOM"] + (["ATOM"] * 4 if C else []) + \
        (["DRANGE"] * 2 if (D and allow_drange) else []) + (["STR"] * 2 if S else [])
    inner = ["NOT", "AND", "OR"] + (["EXISTS", "FORALL", "MIN", "MAX", "EXACT"] * 2 if R else [])
    if depth <= 1 or rng.random() < 0.25:
        k = leaf_kinds[int(rng.integers(len(leaf_kinds)))]
        if k == "ATOM":
            return ("ATOM", int(rng.integers(C)))
        if k == "STR":
            pat = STR_PATTERNS[int(rng.integers(len(STR_PATTERNS)))]
            return ("SEQUAL" if rng.random() < 0.5 else "SCONTAIN", int(rng.integers(S)), pat)
        if k == "DRANGE":
            pool = [-INF, -2.0, -1.5, -0.0, 0.0, 0.5, 1.0, 2.25, 3.0, INF]
            lo = pool[int(rng.integers(len(pool)))]
            hi = pool[int(rng.integers(len(pool)))]
            return ("DRANGE", int(rng.integers(D)), lo, hi)
        return (k,)
    k = inner[int(rng.integers(len(inner)))]
    if k == "NOT":
        return ("NOT", random_tree(rng, shape, depth - 1, n_max, allow_drange))
    if k in ("AND", "OR"):
        m = int(rng.choice([0, 1, 2, 2, 3, 5]))
        return (k, [random_tree(rng, shape, depth - 1, n_max, allow_drange) for _ in range(m)])
    r, inv = int(rng.integers(R)), bool(rng.integers(2))
    child = random_tree(rng, shape, depth - 1, n_max, allow_drange)
    if k in ("EXISTS", "FORALL"):
        return (k, r, inv, child)
    return (k, int(rng.integers(0, n_max + 1)), r, inv, child)


# ------------------------------------------------------------------------------
# C1: enumerated list covering every opcode x {r, r^-} x corner n x ranges


def c1_hypotheses(kb: dict) -> List[tuple]:
    A = [("ATOM", c) for c in range(4)]
    hs: List[tuple] = [("TOP",), ("BOTTOM",), A[0], ("NOT", A[1]), ("NOT", ("NOT", A[2])),
                       ("AND", []), ("OR", []), ("AND", [A[0], A[1]]), ("OR", [A[2], ("NOT", A[3])]),
                       ("AND", [A[0], ("NOT", A[0])]), ("OR", [A[1], ("NOT", A[1])]),
                       ("AND", [A[0], A[1], A[2], A[3], ("NOT", A[0])])]
    maxdeg = 12
    for r in range(2):
        for inv in (False, True):
            hs += [("EXISTS", r, inv, A[r]), ("FORALL", r, inv, A[r + 1]),
                   ("EXISTS", r, inv, ("TOP",)), ("FORALL", r, inv, ("BOTTOM",))]
            for n, k in ((0, "MIN"), (1, "MIN"), (maxdeg, "MIN"), (maxdeg + 1, "MAX"),
                         (1, "MAX"), (0, "MAX"), (2, "EXACT")):
                hs.append((k, n, r, inv, ("OR", [A[(n + r) % 4], ("NOT", A[3])])))
    hs += [("DRANGE", 0, 0.5, 0.5), ("DRANGE", 0, -INF, INF), ("DRANGE", 0, 2.0, 1.0),
           ("DRANGE", 0, 0.0, 0.0), ("DRANGE", 0, -0.0, -0.0), ("DRANGE", 0, INF, INF),
           ("DRANGE", 0, -1.5, 1.0)]
    # depth-3 mixtures
    hs += [("EXISTS", 0, False, ("FORALL", 1, True, ("OR", [A[1], ("NOT", A[2])]))),
           ("AND", [A[0], ("EXISTS", 1, False, ("DRANGE", 0, 0.0, INF))]),
           ("MIN", 2, 0, True, ("AND", [A[2], ("EXISTS", 0, False, ("TOP",))])),
           ("NOT", ("FORALL", 0, False, ("NOT", A[0]))),
           ("OR", [("MAX", 1, 1, False, A[0]), ("EXACT", 0, 0, True, A[3])])]
    while len(hs) < 64:
        hs.append(("EXISTS", len(hs) % 2, bool(len(hs) % 3 == 0), ("AND", [A[len(hs) % 4]])))
    return hs[:64]


# ------------------------------------------------------------------------------
# refinement-style generator (C2 latency set, C4, C5)


class Refiner:
    """One-step downward refinements, SURVEY 8(d) "Refinement-style generator".

    shape: dict(C, R, D); roles: list of role ids usable; data_q: per data
    property a sorted array of quantile bounds; root_concept: optional concept
    every hypothesis starts from (C2: Compound).
    """

    def __init__(self, rng, shape, data_q=None, count_max=16, max_depth=4,
                 card_heavy=False, atoms=None):
        self.rng = rng
        self.C, self.R, self.D = shape["C"], shape["R"], shape["D"]
        self.data_q = data_q or []
        self.count_max = count_max
        self.max_depth = max_depth
        self.card_heavy = card_heavy
        self.atoms = list(range(self.C)) if atoms is None else list(atoms)

    def _r(self):
        return int(self.rng.integers(self.R)), bool(self.rng.integers(2))

    def top_refinement(self):
        """One step down from TOP: A | not A | exists/forall/>=n/<=n rho.TOP | exists d.[q,+inf]."""
        rng = self.rng
        kinds = ["ATOM"] * 6 + ["NATOM"] * 2
        if self.R:
            kinds += ["EXISTS", "EXISTS", "FORALL"] + (["MIN", "MAX"] if not self.card_heavy
                                                        else ["MIN"] * 3 + ["MAX"] * 3)
        if self.D and self.data_q:
            kinds += ["DRANGE"] * (1 if not self.card_heavy else 3)
        k = kinds[int(rng.integers(len(kinds)))]
        if k == "ATOM":
            return ("ATOM", self.atoms[int(rng.integers(len(self.atoms)))])
        if k == "NATOM":
            return ("NOT", ("ATOM", self.atoms[int(rng.integers(len(self.atoms)))]))
        if k == "DRANGE":
            d = int(rng.integers(self.D))
            q = self.data_q[d]
            i = int(rng.integers(len(q)))
            return ("DRANGE", d, float(q[i]), INF)
        r, inv = self._r()
        if k in ("EXISTS", "FORALL"):
            return (k, r, inv, ("TOP",))
        if k == "MIN":
            n = int(rng.integers(0, self.count_max + 1)) if self.card_heavy else int(rng.integers(2, 4))
            return ("MIN", n, r, inv, ("TOP",))
        n = int(rng.integers(0, self.count_max + 1)) if self.card_heavy else int(rng.integers(1, 5))
        return ("MAX", n, r, inv, ("TOP",))

    def refine(self, t, budget_depth):
        """Return one downward refinement of t (depth <= budget_depth) or None."""
        rng = self.rng
        tag = t[0]
        from .format import tree_depth
        for _ in range(6):
            c = self._refine_once(t, budget_depth)
            if c is not None and tree_depth(c) <= budget_depth and c != t:
                return c
        return None

    def _refine_once(self, t, bd):
        rng = self.rng
        tag = t[0]
        if tag == "TOP":
            return self.top_refinement()
        choice = rng.random()
        if tag == "AND":
            if choice < 0.5 and len(t[1]) < 3:
                return ("AND", t[1] + [self.top_refinement()])
            i = int(rng.integers(len(t[1])))
            c = self.refine(t[1][i], bd - 1)
            if c is None:
                return None
            xs = list(t[1])
            if c[0] == "AND":                 # keep conjunctions flat (PAPER.md:521 n-ary op)
                xs[i:i + 1] = c[1]
            else:
                xs[i] = c
            return ("AND", xs) if len(xs) <= 4 else None
        if choice < 0.4 or tag in ("ATOM", "NOT"):
            return ("AND", [t, self.top_refinement()])
        if tag == "EXISTS":
            if rng.random() < 0.25:
                return ("MIN", 2, t[1], t[2], t[3])
            c = self.refine(t[3], bd - 1)
            return None if c is None else ("EXISTS", t[1], t[2], c)
        if tag == "FORALL":
            c = self.refine(t[3], bd - 1)
            return None if c is None else ("FORALL", t[1], t[2], c)
        if tag == "MIN":
            if rng.random() < 0.4 and t[1] < self.count_max:
                return ("MIN", t[1] + 1, t[2], t[3], t[4])
            c = self.refine(t[4], bd - 1)
            return None if c is None else ("MIN", t[1], t[2], t[3], c)
        if tag == "MAX":
            if rng.random() < 0.4 and t[1] > 0:
                return ("MAX", t[1] - 1, t[2], t[3], t[4])
            c = self.refine(t[4], bd - 1)
            return None if c is None else ("MAX", t[1], t[2], t[3], c)
        if tag == "DRANGE":
            q = self.data_q[t[1]]
            i = int(np.searchsorted(q, t[2]))
            if math.isinf(t[3]) and i + 1 < len(q) and rng.random() < 0.5:
                return ("DRANGE", t[1], float(q[i + 1]), INF)
            j = int(rng.integers(i, len(q)))
            return ("DRANGE", t[1], t[2], float(q[j]))
        return ("AND", [t, self.top_refinement()])


def refinement_batch(seed: int, shape: dict, n_hyps: int, data_q=None, children: int = 8,
                     max_depth: int = 4, card_heavy: bool = False, root=None,
                     count_max: int = 16, atoms=None) -> List[tuple]:
    """Beam/BFS from TOP (or `root`): each parent emits up to `children` contiguous refinements."""
    rng = np.random.default_rng(seed)
    ref = Refiner(rng, shape, data_q, count_max=count_max, max_depth=max_depth,
                  card_heavy=card_heavy, atoms=atoms)
    start = root if root is not None else ("TOP",)
    out: List[tuple] = []
    frontier = [start]
    seen = set()
    while len(out) < n_hyps and frontier:
        nxt = []
        for p in frontier:
            for _ in range(children):
                c = ref.refine(p, max_depth)
                if c is None:
                    continue
                if card_heavy and not _has_card_or_range(c):
                    c = ("AND", [c, ref.top_refinement()]) if c[0] != "AND" else c
                    if not _has_card_or_range(c):
                        continue
                key = repr(c)
                if key in seen:
                    continue
                seen.add(key)
                out.append(c)
                nxt.append(c)
                if len(out) >= n_hyps:
                    break
            if len(out) >= n_hyps:
                break
        if not nxt:
            break
        rng.shuffle(nxt)
        frontier = nxt
    return out[:n_hyps]


def _has_card_or_range(t) -> bool:
    tag = t[0]
    if tag in ("MIN", "MAX", "EXACT", "DRANGE"):
        return True
    if tag in ("AND", "OR"):
        return any(_has_card_or_range(c) for c in t[1])
    if tag == "NOT":
        return _has_card_or_range(t[1])
    if tag in ("EXISTS", "FORALL"):
        return _has_card_or_range(t[3])
    return False


def data_quantiles(kb: dict, d: int = 0, qs=(0.5, 0.7, 0.8, 0.9, 0.95, 0.99)) -> np.ndarray:
    lo, hi = int(kb["data_off"][d]), int(kb["data_off"][d + 1])
    v = kb["data_val"][lo:hi]
    v = v[~np.isnan(v)]
    if len(v) == 0:
        return np.zeros(0, np.float32)
    return np.unique(np.quantile(v, qs).astype(np.float32))


def c2_hypotheses(kb: dict, n: int = 256, seed: int = 2) -> List[tuple]:
    """256 depth-4 refinements rooted at Compound."""
    names = kb["names"]["concepts"]
    comp = names.index("Compound")
    shape = {"C": len(names), "R": 3, "D": 1}
    hs = refinement_batch(seed, shape, 4 * n, data_q=[data_quantiles(kb, 0, (0.1, 0.3, 0.5, 0.7, 0.9))],
                          children=6, max_depth=4, root=("AND", [("ATOM", comp)]),
                          atoms=list(range(1, len(names))))
    from .format import tree_depth
    deep = [h for h in hs if tree_depth(h) == 4]
    rest = [h for h in hs if tree_depth(h) != 4]
    return (deep + rest)[:n]


def c3_hypotheses() -> List[tuple]:
    """8 fixed single hypotheses, nested exists/forall + inverse (r=role 0, s=role 1)."""
    A = lambda i: ("ATOM", i)
    r, s = 0, 1
    return [
        ("EXISTS", r, False, ("AND", [A(1), ("FORALL", s, True, ("OR", [A(2), ("NOT", A(3))]))])),  # H3a
        ("MIN", 2, r, True, ("EXISTS", s, False, A(4))),                                             # H3b
        ("FORALL", r, False, ("OR", [("EXISTS", r, False, A(5)), ("DRANGE", 0, 0.5, INF)])),       # H3c
        ("AND", [A(6), ("EXISTS", s, True, ("EXISTS", r, False, A(7)))]),
        ("MAX", 3, r, False, ("AND", [A(8), ("NOT", A(9))])),
        ("EXISTS", r, True, ("FORALL", r, False, ("EXISTS", s, False, ("TOP",)))),
        ("OR", [("EXACT", 1, s, False, A(10)), ("FORALL", s, True, ("BOTTOM",))]),
        ("AND", [("EXISTS", r, False, A(11)), ("EXISTS", s, True, ("NOT", A(12))),
                 ("DRANGE", 0, -1.0, 1.0)]),
    ]


def c4_hypotheses(kb: dict, n: int = 1_000_000, seed: int = 4) -> List[tuple]:
    shape = {"C": int(kb["concept_bits"].shape[0]), "R": len(kb["role_edge_off"]) - 1,
             "D": len(kb["data_off"]) - 1}
    return refinement_batch(seed, shape, n, data_q=[data_quantiles(kb)], children=8, max_depth=4)


def c5_hypotheses(kb: dict, n: int = 100_000, seed: int = 5) -> List[tuple]:
    shape = {"C": int(kb["concept_bits"].shape[0]), "R": len(kb["role_edge_off"]) - 1,
             "D": len(kb["data_off"]) - 1}
    q = data_quantiles(kb, 0, tuple(np.linspace(0.5, 0.99, 12)))
    return refinement_batch(seed, shape, n, data_q=[q], children=8, max_depth=4,
                            card_heavy=True, count_max=16)


# ------------------------------------------------------------------------------
# parallel generation of large batches as flat arrays


def _gen_chunk(args):
    kind, shape, data_q, n, seed = args
    from .format import flatten
    if kind == "c4":
        hs = refinement_batch(seed, shape, n, data_q=data_q, children=8, max_depth=4)
    elif kind == "c5":
        hs = refinement_batch(seed, shape, n, data_q=data_q, children=8, max_depth=4,
                              card_heavy=True, count_max=16)
    else:
        raise ValueError(kind)
    return flatten(hs)


def concat_arrays(parts):
    """Concatenate several (nodes, child_idx, roots) triples into one."""
    from .format import NODE_DTYPE, OP_NAMES, NodeArray, node_patterns
    nodes_l, kids_l, roots_l, pats = [], [], [], []
    n_off = k_off = 0
    s_ops = np.array([OP_NAMES.index("SEQUAL"), OP_NAMES.index("SCONTAIN")], dtype=np.uint8)
    for nodes, kids, roots in parts:
        nd = np.asarray(nodes).copy()
        nd["child_begin"] += np.uint32(k_off)
        p = node_patterns(nodes)
        if p:
            nd["n"][np.isin(nd["op"], s_ops)] += np.uint32(len(pats))
            pats += p
        nodes_l.append(nd)
        kids_l.append(kids + np.uint32(n_off))
        roots_l.append(roots + np.uint32(n_off))
        n_off += len(nodes)
        k_off += len(kids)
    if not parts:
        return np.zeros(0, NODE_DTYPE), np.zeros(0, np.uint32), np.zeros(0, np.uint32)
    nodes = np.concatenate(nodes_l).view(NodeArray)
    nodes.patterns = pats
    return nodes, np.concatenate(kids_l), np.concatenate(roots_l)


def batch_arrays(kind: str, kb: dict, n: int, seed: int, chunk: int = 25_000,
                 workers: Optional[int] = None, first_chunk: int = 0):
    """Generate a C4/C5-style batch of n hypotheses as flat ABI arrays.

    The batch is cut into independent beams of `chunk` hypotheses (seed
    (seed, i)); each beam keeps its sibling families contiguous.  `first_chunk` starts
    at beam i = first_chunk, so a rank can generate just its own slice of a larger batch.
    """
    import os
    from concurrent.futures import ProcessPoolExecutor
    shape = {"C": int(kb["concept_bits"].shape[0]), "R": len(kb["role_edge_off"]) - 1,
             "D": len(kb["data_off"]) - 1}
    if kind == "c4":
        dq = [data_quantiles(kb)]
    else:
        dq = [data_quantiles(kb, 0, tuple(np.linspace(0.5, 0.99, 12)))]
    jobs = []
    i = 0
    while i * chunk < n:
        jobs.append((kind, shape, dq, min(chunk, n - i * chunk), int(seed) * 100003 + first_chunk + i))
        i += 1
    workers = workers or min(len(jobs), os.cpu_count() or 1, 32)
    if workers <= 1 or len(jobs) == 1:
        parts = [_gen_chunk(j) for j in jobs]
    else:
        import multiprocessing as mp
        with ProcessPoolExecutor(workers, mp_context=mp.get_context("fork")) as ex:
            parts = list(ex.map(_gen_chunk, jobs))
    return concat_arrays(parts)


def string_hypotheses(kb: dict, n: int = 400, seed: int = 7) -> List[tuple]:
    """Hypotheses over a string_kb: EQUAL on asserted values (hits) and on absent values
    (the PAPER.md:457 short-circuit), CONTAIN on substrings of asserted values, on
    absent substrings and on whole values, alone and composed with the other constructors."""
    rng = np.random.default_rng(seed)
    vocab = kb["_vocab"]
    S = len(kb["str_off"]) - 1
    R = len(kb["role_edge_off"]) - 1
    C = kb["concept_bits"].shape[0]

    def leaf():
        s = int(rng.integers(S))
        v = vocab[int(rng.integers(min(len(vocab), 50)))] if rng.random() < 0.5 else vocab[int(rng.integers(len(vocab)))]
        u = rng.random()
        if u < 0.3:
            return ("SEQUAL", s, v)
        if u < 0.4:
            return ("SEQUAL", s, v + b"#absent")
        if u < 0.85:
            a = int(rng.integers(len(v)))
            b = int(rng.integers(a + 1, len(v) + 1))
            return ("SCONTAIN", s, v[a:b])
        return ("SCONTAIN", s, b"#" + v[:3])

    out = []
    for _ in range(n):
        k = int(rng.integers(6))
        if k == 0:
            t = leaf()
        elif k == 1:
            t = ("AND", [("ATOM", int(rng.integers(C))), leaf()])
        elif k == 2:
            t = ("OR", [leaf(), leaf()])
        elif k == 3:
            t = ("NOT", leaf())
        elif k == 4 and R:
            t = ("EXISTS", int(rng.integers(R)), bool(rng.integers(2)), leaf())
        else:
            t = ("AND", [("NOT", ("ATOM", int(rng.integers(C)))), ("OR", [leaf(), ("ATOM", 0)])])
        out.append(t)
    return out
