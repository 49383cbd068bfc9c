"""Input formats shared by the generators, the oracle and the C-ABI binding.

This module holds *formats only* (record layouts, opcode numbers, a tree
flattener and an s-expression reader).  It contains none of the method's
arithmetic: no set operation, no restriction, no coverage count.  Both the
oracle (`oracle/`) and the product binding (`paper_2412_00802_b200/`) read the
arrays produced here; neither imports the other.

Opcode numbers and the node record mirror `include/hedl.h` (the ABI) and the
constructor list of the paper's ALCQI(D) language (§III;
operators §III-B, Algs. 1-10).
"""
from __future__ import annotations

import math
import re
from typing import Dict, List, Sequence, Tuple

import numpy as np

# ---- opcodes (== hedl.h HEDL_OP_*) -----------------------------------------
TOP, BOTTOM, ATOM, NOT, AND, OR, EXISTS, FORALL, MIN, MAX, EXACT, DRANGE, SEQUAL, SCONTAIN = range(14)
OP_NAMES = ["TOP", "BOTTOM", "ATOM", "NOT", "AND", "OR", "EXISTS", "FORALL",
            "MIN", "MAX", "EXACT", "DRANGE", "SEQUAL", "SCONTAIN"]
ROLE_OPS = (EXISTS, FORALL, MIN, MAX, EXACT)
COUNT_OPS = (MIN, MAX, EXACT)

FLAG_INV = 1  # node.flags bit: role is the inverse r^- (§III-B2)

# compile flags (== hedl.h HEDL_COMPILE_*)
COMPILE_NO_CSE = 1
COMPILE_NO_REWRITE = 2
COMPILE_COMPAT_PAPER_MAX = 4

# hedl_node {u8 op; u8 flags; u16 pad; u32 arg; u32 n; f32 lo, hi; u32 child_begin, child_count}
NODE_DTYPE = np.dtype([
    ("op", np.uint8), ("flags", np.uint8), ("pad", np.uint16),
    ("arg", np.uint32), ("n", np.uint32),
    ("lo", np.float32), ("hi", np.float32),
    ("child_begin", np.uint32), ("child_count", np.uint32),
], align=True)
assert NODE_DTYPE.itemsize == 28


def string_fields(kb: dict):
    """The string concrete-role arrays of a KB dict (empty when the KB has none)."""
    if "str_off" in kb:
        return (np.asarray(kb["str_off"], np.uint64), np.asarray(kb["str_subj"], np.uint32),
                np.asarray(kb["str_val_off"], np.uint64), np.asarray(kb["str_bytes"], np.uint8))
    return (np.zeros(1, np.uint64), np.zeros(0, np.uint32), np.zeros(1, np.uint64), np.zeros(0, np.uint8))


def words(n_individuals: int) -> int:
    """W = ceil(N/32): u32 words of one LSB-first bitset row."""
    return (n_individuals + 31) // 32


# ---- trees -------------------------------------------------------------------
# A hypothesis tree is a nested tuple:
#   ("TOP",) ("BOTTOM",) ("ATOM", c) ("NOT", t) ("AND", [t..]) ("OR", [t..])
#   ("EXISTS", r, inv, t) ("FORALL", r, inv, t)
#   ("MIN", n, r, inv, t) ("MAX", n, r, inv, t) ("EXACT", n, r, inv, t)
#   ("DRANGE", d, lo, hi)

class NodeArray(np.ndarray):
    """A NODE_DTYPE array that carries its string-pattern table (`.patterns`, list of bytes,
    indexed by node.n of SEQUAL / SCONTAIN nodes) through unpacking and slicing."""

    def __array_finalize__(self, obj):
        self.patterns = getattr(obj, "patterns", [])


def node_patterns(nodes) -> list:
    return list(getattr(nodes, "patterns", []) or [])


class Flat(tuple):
    """(nodes, child_idx, roots); `.patterns` = string-restriction patterns (list of bytes)
    referenced by SEQUAL / SCONTAIN nodes through node.n (the hedl_patterns table)."""

    @property
    def patterns(self):
        return node_patterns(self[0])


def flatten(trees: Sequence[tuple], share: bool = False):
    """Post-order flatten trees into (nodes, child_idx, roots) arrays.

    With share=True, structurally identical subtrees are emitted once (the ABI
    accepts DAGs); the default emits every occurrence so that the compiler's
    own common-subexpression elimination is what gets exercised.
    """
    recs: List[tuple] = []
    kids: List[int] = []
    memo: Dict[tuple, int] = {}
    patterns: List[bytes] = []

    def emit(t) -> int:
        if share:
            key = _freeze(t)
            if key in memo:
                return memo[key]
        tag = t[0]
        op = OP_NAMES.index(tag)
        flags, arg, n, lo, hi, ch = 0, 0, 0, 0.0, 0.0, []
        if tag in ("TOP", "BOTTOM"):
            pass
        elif tag == "ATOM":
            arg = t[1]
        elif tag == "NOT":
            ch = [emit(t[1])]
        elif tag in ("AND", "OR"):
            ch = [emit(c) for c in t[1]]
        elif tag in ("EXISTS", "FORALL"):
            arg, flags, ch = t[1], (FLAG_INV if t[2] else 0), [emit(t[3])]
        elif tag in ("MIN", "MAX", "EXACT"):
            n, arg, flags, ch = t[1], t[2], (FLAG_INV if t[3] else 0), [emit(t[4])]
        elif tag == "DRANGE":
            arg, lo, hi = t[1], t[2], t[3]
        elif tag in ("SEQUAL", "SCONTAIN"):            # (tag, string role, pattern)
            arg = t[1]
            pat = t[2].encode() if isinstance(t[2], str) else bytes(t[2])
            n = len(patterns)
            patterns.append(pat)
        else:
            raise ValueError(tag)
        begin = len(kids)
        kids.extend(ch)
        recs.append((op, flags, 0, arg, n, lo, hi, begin, len(ch)))
        idx = len(recs) - 1
        if share:
            memo[key] = idx
        return idx

    roots = [emit(t) for t in trees]
    nodes = (np.array(recs, dtype=NODE_DTYPE) if recs else np.zeros(0, NODE_DTYPE)).view(NodeArray)
    nodes.patterns = patterns
    return Flat((nodes, np.array(kids, dtype=np.uint32), np.array(roots, dtype=np.uint32)))


def pack_strings(strs: Sequence[bytes]):
    """Byte strings -> (offsets u64[n+1], blob u8[]) (the hedl_patterns / string-value layout)."""
    off = np.zeros(len(strs) + 1, dtype=np.uint64)
    for i, b in enumerate(strs):
        off[i + 1] = off[i] + len(b)
    blob = np.frombuffer(b"".join(strs), dtype=np.uint8).copy() if strs else np.zeros(0, np.uint8)
    return off, blob


def _freeze(t):
    if isinstance(t, (list, tuple)):
        return tuple(_freeze(x) for x in t)
    if isinstance(t, float):
        return ("f", np.float32(t).tobytes())
    return t


def tree_depth(t) -> int:
    """Depth per SURVEY Q16: literals (A, not A, TOP, BOTTOM, DRANGE) are 1."""
    tag = t[0]
    if tag in ("TOP", "BOTTOM", "ATOM", "DRANGE", "SEQUAL", "SCONTAIN"):
        return 1
    if tag == "NOT":
        return 1 if t[1][0] == "ATOM" else 1 + tree_depth(t[1])
    if tag in ("AND", "OR"):
        return 1 + max((tree_depth(c) for c in t[1]), default=0)
    return 1 + tree_depth(t[-1])


def tree_to_text(t, names=None) -> str:
    cn = (names or {}).get("concepts")
    rn = (names or {}).get("roles")
    dn = (names or {}).get("data")
    tag = t[0]

    def role(r, inv):
        s = rn[r] if rn else f"r{r}"
        return f"(INV {s})" if inv else s

    if tag in ("TOP", "BOTTOM"):
        return tag
    if tag == "ATOM":
        return cn[t[1]] if cn else f"A{t[1]}"
    if tag == "NOT":
        return f"(NOT {tree_to_text(t[1], names)})"
    if tag in ("AND", "OR"):
        return "(" + " ".join([tag] + [tree_to_text(c, names) for c in t[1]]) + ")"
    if tag == "EXISTS":
        return f"(SOME {role(t[1], t[2])} {tree_to_text(t[3], names)})"
    if tag == "FORALL":
        return f"(ONLY {role(t[1], t[2])} {tree_to_text(t[3], names)})"
    if tag in ("MIN", "MAX", "EXACT"):
        kw = {"MIN": "MIN", "MAX": "MAX", "EXACT": "EXACTLY"}[tag]
        return f"({kw} {t[1]} {role(t[2], t[3])} {tree_to_text(t[4], names)})"
    if tag == "DRANGE":
        d = dn[t[1]] if dn else f"d{t[1]}"
        return f"(DRANGE {d} {_fmt(t[2])} {_fmt(t[3])})"
    if tag in ("SEQUAL", "SCONTAIN"):
        sn = (names or {}).get("strings")
        sr = sn[t[1]] if sn else f"s{t[1]}"
        pat = t[2] if isinstance(t[2], str) else bytes(t[2]).decode("utf-8", "backslashreplace")
        return f'(SSOME {sr} {"EQUAL" if tag == "SEQUAL" else "CONTAIN"} "{_esc(pat)}")'
    raise ValueError(tag)


def _esc(s: str) -> str:
    return s.replace("\\", "\\\\").replace('"', '\\"')


def _fmt(x: float) -> str:
    if math.isinf(x):
        return "+inf" if x > 0 else "-inf"
    return repr(float(np.float32(x)))


# ---- s-expression reader (SPEC.md:347-355 grammar, extended per SURVEY 8(b)) --
_TOK = re.compile(r'"(?:[^"\\]|\\.)*"|\(|\)|[^\s()]+')


def parse(text: str, names) -> tuple:
    """Parse one hypothesis in the s-expression grammar into a tree.

    `names` maps "concepts"/"roles"/"data" to lists of names.  Extensions over
    SPEC.md:347-355: TOP, BOTTOM, (NOT e) for any e, (DRANGE d lo hi) with
    closed float32 bounds, (INV r) nesting ((INV (INV r)) == r).
    """
    toks = _TOK.findall(text)
    pos = [0]
    cidx = {s: i for i, s in enumerate(names.get("concepts", []))}
    ridx = {s: i for i, s in enumerate(names.get("roles", []))}
    didx = {s: i for i, s in enumerate(names.get("data", []))}
    sidx = {s: i for i, s in enumerate(names.get("strings", []))}

    def nxt():
        if pos[0] >= len(toks):
            raise SyntaxError("unexpected end of hypothesis")
        t = toks[pos[0]]
        pos[0] += 1
        return t

    def expect(s):
        t = nxt()
        if t != s:
            raise SyntaxError(f"expected {s!r}, got {t!r}")

    def role():
        t = nxt()
        if t == "(":
            expect("INV")
            r, inv = role()
            expect(")")
            return r, not inv
        if t not in ridx:
            raise KeyError(f"unknown role {t!r}")
        return ridx[t], False

    def num(t):
        v = float(t)
        if math.isnan(v):
            raise ValueError("NaN bound")
        return float(np.float32(v))

    def expr():
        t = nxt()
        if t == "TOP":
            return ("TOP",)
        if t == "BOTTOM":
            return ("BOTTOM",)
        if t != "(":
            if t not in cidx:
                raise KeyError(f"unknown concept {t!r}")
            return ("ATOM", cidx[t])
        kw = nxt()
        if kw == "NOT":
            e = ("NOT", expr())
        elif kw in ("AND", "OR"):
            xs = []
            while toks[pos[0]] != ")":
                xs.append(expr())
            e = (kw, xs)
        elif kw in ("SOME", "ONLY"):
            r, inv = role()
            e = ("EXISTS" if kw == "SOME" else "FORALL", r, inv, expr())
        elif kw in ("MIN", "MAX", "EXACTLY"):
            n = int(nxt())
            if n < 0:
                raise ValueError("negative cardinality")
            r, inv = role()
            e = ({"MIN": "MIN", "MAX": "MAX", "EXACTLY": "EXACT"}[kw], n, r, inv, expr())
        elif kw == "DRANGE":
            d = nxt()
            if d not in didx:
                raise KeyError(f"unknown data property {d!r}")
            e = ("DRANGE", didx[d], num(nxt()), num(nxt()))
        elif kw == "SSOME":                       # SPEC.md:353 string restrictions
            sr = nxt()
            if sr not in sidx:
                raise KeyError(f"unknown string role {sr!r}")
            mode = nxt()
            lit = nxt()
            if not (lit.startswith('"') and lit.endswith('"')):
                raise SyntaxError("string literal expected")
            val = re.sub(r"\\(.)", r"\1", lit[1:-1])
            if mode not in ("EQUAL", "CONTAIN"):
                raise SyntaxError(f"unknown string restriction {mode!r}")
            e = ("SEQUAL" if mode == "EQUAL" else "SCONTAIN", sidx[sr], val)
        else:
            raise SyntaxError(f"unknown constructor {kw!r}")
        expect(")")
        return e

    e = expr()
    if pos[0] != len(toks):
        raise SyntaxError("trailing tokens")
    return e


# ---- KB dict helpers -----------------------------------------------------------

def kb_from_sets(n: int, concepts: Sequence[Sequence[int]],
                 roles: Sequence[Sequence[Tuple[int, int]]],
                 data: Sequence[Sequence[Tuple[int, float]]],
                 pos: Sequence[int], neg: Sequence[int],
                 strings: Sequence[Sequence[Tuple[int, bytes]]] = ()) -> dict:
    """Assemble a KB dict (the hedl_kb_desc arrays) from explicit member lists.

    Packing a member list into LSB-first words is the input format itself
    (bit i&31 of word i>>5), not a step of the method.
    """
    w = words(n)
    cb = np.zeros((len(concepts), w), dtype=np.uint32)
    for c, mem in enumerate(concepts):
        for i in mem:
            cb[c, i >> 5] |= np.uint32(1) << np.uint32(i & 31)
    off = [0]
    subj, obj = [], []
    for pairs in roles:
        for s, o in pairs:
            subj.append(s)
            obj.append(o)
        off.append(len(subj))
    doff = [0]
    dsubj, dval = [], []
    for pairs in data:
        for s, v in pairs:
            dsubj.append(s)
            dval.append(v)
        doff.append(len(dsubj))
    soff, ssubj, svals = [0], [], []
    for pairs in strings:
        for s_, v in pairs:
            ssubj.append(s_)
            svals.append(v.encode() if isinstance(v, str) else bytes(v))
        soff.append(len(ssubj))
    vo, blob = pack_strings(svals)
    return {
        "str_off": np.array(soff, dtype=np.uint64),
        "str_subj": np.array(ssubj, dtype=np.uint32),
        "str_val_off": vo,
        "str_bytes": blob,
        "N": n,
        "concept_bits": cb,
        "role_edge_off": np.array(off, dtype=np.uint64),
        "edge_subj": np.array(subj, dtype=np.uint32),
        "edge_obj": np.array(obj, dtype=np.uint32),
        "data_off": np.array(doff, dtype=np.uint64),
        "data_subj": np.array(dsubj, dtype=np.uint32),
        "data_val": np.array(dval, dtype=np.float32),
        "pos_ids": np.array(sorted(pos), dtype=np.uint32),
        "neg_ids": np.array(sorted(neg), dtype=np.uint32),
    }
