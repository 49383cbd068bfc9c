"""Pure-Python brute-force oracle for tiny KBs (N <= 64).

ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every quantifier ranges over all of Delta = {0..N-1} (never over adjacency),
following the textbook ALCQI(D) semantics the paper implements under CWA /
UNA (§III-A):

  TOP -> Delta; BOTTOM -> {}; A -> A^I; NOT C -> Delta minus C
  AND/OR -> intersection/union (empty AND = Delta, empty OR = {}; Alg. 1 init)
  exists rho.C -> {x | some y in Delta: (x,y) in rho and y in C}
  forall rho.C -> {x | every y in Delta: (x,y) in rho implies y in C}
  >=n/<=n/=n rho.C -> {x | #{y in Delta: (x,y) in rho, y in C} >= / <= / == n}
  exists d.[lo,hi] -> {x | some asserted (x,v): lo <= v <= hi} in float32
  EQUAL s v   -> {x | some asserted (x,w) of s: w == v}      (Alg. 11)
  CONTAIN s v -> {x | some asserted (x,w) of s: v substring of w}  (Alg. 13; empty v rejected)
  r^- = {(y,x) | (x,y) in r}.
"""
from __future__ import annotations

import numpy as np

_OPS = ["TOP", "BOTTOM", "ATOM", "NOT", "AND", "OR", "EXISTS", "FORALL", "MIN", "MAX",
        "EXACT", "DRANGE", "SEQUAL", "SCONTAIN"]


def _members(words, n):
    return {i for i in range(n) if (int(words[i // 32]) >> (i % 32)) & 1}


class BruteKB:
    def __init__(self, kb: dict):
        n = int(kb["N"])
        assert n <= 64, "brute force is for tiny KBs only"
        self.N = n
        self.delta = set(range(n))
        cb = np.asarray(kb["concept_bits"])
        self.concepts = [_members(cb[c], n) for c in range(cb.shape[0])] if cb.size else \
            [set() for _ in range(cb.shape[0] if cb.ndim == 2 else 0)]
        off = [int(v) for v in kb["role_edge_off"]]
        es, eo = kb["edge_subj"], kb["edge_obj"]
        self.roles = [set(zip(es[off[r]:off[r + 1]].tolist(), eo[off[r]:off[r + 1]].tolist()))
                      for r in range(len(off) - 1)]
        doff = [int(v) for v in kb["data_off"]]
        ds, dv = kb["data_subj"], np.asarray(kb["data_val"], dtype=np.float32)
        self.data = [list(zip(ds[doff[d]:doff[d + 1]].tolist(), dv[doff[d]:doff[d + 1]]))
                     for d in range(len(doff) - 1)]
        from synth.format import string_fields
        so, ss, sv, sb = string_fields(kb)
        blob = bytes(sb)
        self.strings = [[(int(ss[k]), blob[int(sv[k]):int(sv[k + 1])]) for k in range(int(so[r]), int(so[r + 1]))]
                        for r in range(len(so) - 1)]
        self.pos = set(int(i) for i in kb["pos_ids"])
        self.neg = set(int(i) for i in kb["neg_ids"])

    def role(self, r, inv):
        rel = self.roles[r]
        return {(y, x) for (x, y) in rel} if inv else rel

    def eval(self, nodes, kids, i, compat_paper_max=False, patterns=()):
        nd = nodes[i]
        op = _OPS[int(nd["op"])]
        ch = [int(k) for k in kids[int(nd["child_begin"]):int(nd["child_begin"]) + int(nd["child_count"])]]
        D = self.delta
        ev = lambda j: self.eval(nodes, kids, j, compat_paper_max, patterns)
        if op == "TOP":
            return set(D)
        if op == "BOTTOM":
            return set()
        if op == "ATOM":
            return set(self.concepts[int(nd["arg"])])
        if op == "NOT":
            return D - ev(ch[0])
        if op == "AND":
            out = set(D)
            for j in ch:
                out &= ev(j)
            return out
        if op == "OR":
            out = set()
            for j in ch:
                out |= ev(j)
            return out
        if op in ("SEQUAL", "SCONTAIN"):
            pat = patterns[int(nd["n"])]
            if op == "SCONTAIN" and not pat:
                raise ValueError("empty CONTAIN pattern")
            hit = (lambda w: w == pat) if op == "SEQUAL" else (lambda w: pat in w)
            return {x for x in D if any(s == x and hit(w) for (s, w) in self.strings[int(nd["arg"])])}
        if op == "DRANGE":
            lo, hi = np.float32(nd["lo"]), np.float32(nd["hi"])
            return {x for x in D if any(s == x and lo <= v <= hi for (s, v) in self.data[int(nd["arg"])])}
        rho = self.role(int(nd["arg"]), bool(int(nd["flags"]) & 1))
        c = ev(ch[0])
        n = int(nd["n"])
        if op == "EXISTS":
            return {x for x in D if any((x, y) in rho and y in c for y in D)}
        if op == "FORALL":
            return {x for x in D if all(((x, y) not in rho) or (y in c) for y in D)}
        cnt = {x: sum(1 for y in D if (x, y) in rho and y in c) for x in D}
        if op == "MIN":
            return {x for x in D if cnt[x] >= n}
        if op == "EXACT":
            return {x for x in D if cnt[x] == n}
        if compat_paper_max:
            return {x for x in D if 0 < cnt[x] <= n}
        return {x for x in D if cnt[x] <= n}

    def coverage(self, h):
        tp, fp = len(h & self.pos), len(h & self.neg)
        return tp, fp, len(self.pos) - tp, len(self.neg) - fp


def evaluate(kb: dict, nodes, child_idx, roots, compat_paper_max=False, patterns=None):
    """-> list of (instance set, (tp, fp, fn, tn)) per root."""
    if patterns is None:
        patterns = list(getattr(nodes, "patterns", []) or [])
    b = BruteKB(kb)
    out = []
    for r in roots:
        h = b.eval(nodes, child_idx, int(r), compat_paper_max, patterns)
        out.append((h, b.coverage(h)))
    return out


def to_words(members, n):
    w = np.zeros((n + 31) // 32, dtype=np.uint32)
    for i in members:
        w[i // 32] |= np.uint32(1 << (i % 32))
    return w
