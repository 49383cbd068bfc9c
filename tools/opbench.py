"""Operator micro-benchmarks mirroring the paper's Tables 2, 4, card_role and 8.

Paper setup: conjunction / disjunction of 5 concepts over 10..10^7
individuals and of 1..32 concepts over 10^6 (Table 2); exists / forall over the
"single subject" (one hub) and "unique subject" (degree <= 1) regimes with 10..10^7
assertions (Table 4); MIN / MAX cardinality (card_role table); numeric
existential restriction with every value one constant and the string EQUAL / CONTAIN rows
(Table 8; plus a distinct-values variant of ours, where interning cannot
collapse the assertions).

For each cell: the hypothesis is compiled once, then
  * latency_us : host wall time of hedl_eval_one (entry -> counts on the host), median of reps;
  * kernel_us  : device time of the library's kernels for that call (CUDA events), median;
and every cell is checked against the oracle (bit-exact bitset and counts, counts-only rows on
their counts), the paper's 10^7 sizes included.
Writes a JSON list to argv[1] (default profiles/opbench.json) and prints a markdown table with the
paper's GTX 970 column beside ours (context only: other hardware, byte memberships).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2412_00802_b200 as hedl  # noqa: E402
from oracle import setsem  # noqa: E402
from synth import abox  # noqa: E402
from synth.format import flatten, kb_from_sets  # noqa: E402

# paper GPU (GTX 970) microseconds, Tables 2/4/card/8 (context)
PAPER_GPU = {
    ("and5", 10): 15, ("and5", 100): 15, ("and5", 1000): 15, ("and5", 10000): 16, ("and5", 100000): 26,
    ("and5", 1000000): 137, ("and5", 10000000): 1208,
    ("or5", 1000000): 135, ("or5", 10000000): 1198,
    ("exists_unique", 10000000): 1317, ("exists_single", 10000000): 1189,
    ("forall_unique", 10000000): 1312, ("forall_single", 10000000): 1189,
    ("min_unique", 10000000): 2190, ("min_single", 10000000): 10525,
    ("max_unique", 10000000): 2191, ("max_single", 10000000): 10584,
    ("num_unique", 10000000): 1184, ("num_single", 10000000): 1042,
    ("str_equal_single", 10000000): 957, ("str_contain_single", 10000000): 2346,
    ("str_equal_unique", 10000000): 1102, ("str_contain_unique", 10000000): 12551,
    ("str_equal_single", 1000000): 126, ("str_contain_single", 1000000): 287,
    ("str_equal_unique", 1000000): 134, ("str_contain_unique", 1000000): 1459,
}


def concepts_kb(n, k, seed):
    rng = np.random.default_rng(seed)
    w = (n + 31) // 32
    cb = np.zeros((k, w), dtype=np.uint32)
    for c in range(k):
        b = np.zeros(w * 32, dtype=bool)
        b[:n] = rng.random(n) < 0.5
        cb[c] = np.packbits(b, bitorder="little").view("<u4")
    perm = rng.permutation(n)
    m = max(1, n // 100)
    return {"N": n, "concept_bits": cb, "role_edge_off": np.zeros(1, np.uint64),
            "edge_subj": np.zeros(0, np.uint32), "edge_obj": np.zeros(0, np.uint32),
            "data_off": np.zeros(1, np.uint64), "data_subj": np.zeros(0, np.uint32),
            "data_val": np.zeros(0, np.float32),
            "pos_ids": np.sort(perm[:m]).astype(np.uint32), "neg_ids": np.sort(perm[m:2 * m]).astype(np.uint32)}


def measure(kb_np, tree, reps, check, bits=True):
    """bits=True: the instance bitset is produced (full-row work, as the paper's operators);
    bits=False: counts only (root conjunctions run on example-projected rows)."""
    import torch
    k = hedl.hedl_kb_load(kb_np, 0)
    nodes, kids, roots = flatten([tree])      # nodes carry the string-pattern table
    prog = hedl.hedl_compile(k, nodes, kids, roots)
    for _ in range(3):
        hedl.hedl_eval_one(k, prog, 0, want_bits=bits)
    lat, ker = [], []
    for _ in range(reps):
        hedl.prof_reset()
        hedl.prof_enable(True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, c = hedl.hedl_eval_one(k, prog, 0, want_bits=bits)
        lat.append(time.perf_counter() - t0)
        hedl.prof_enable(False)
        ker.append(sum(e["total_ms"] for e in hedl.prof_read()))
    ok = None
    if check:
        # the measured call's counts (bits or counts-only path) and the full bitset, vs the oracle
        ob, oc = setsem.evaluate(kb_np, nodes, kids, roots, threads=os.cpu_count())
        want = tuple(int(v) for v in oc[0])
        b, c1 = hedl.hedl_eval_one(k, prog, 0, want_bits=True)
        ok = bool(np.array_equal(b.cpu().numpy().view(np.uint32), ob[0]) and c1 == want and c == want)
    prog.free()
    k.free()
    return float(np.median(lat)) * 1e6, float(np.median(ker)) * 1e3, ok


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "opbench.json")
    quick = "--quick" in sys.argv
    rows = []
    sizes = [10, 100, 1000, 10_000, 100_000, 1_000_000, 10_000_000]
    if quick:
        sizes = [1000, 1_000_000]
    A = lambda i: ("ATOM", i)
    for n in sizes:                                            # Table 2: 5 concepts, varying N
        kb = concepts_kb(n, 5, n)
        for name, tree in (("and5", ("AND", [A(i) for i in range(5)])), ("or5", ("OR", [A(i) for i in range(5)]))):
            lat, ker, ok = measure(kb, tree, 30, True)
            rows.append({"op": name, "size": n, "latency_us": lat, "kernel_us": ker, "parity": ok,
                         "paper_gtx970_us": PAPER_GPU.get((name, n))})
            lat, ker, ok = measure(kb, tree, 30, True, bits=False)
            rows.append({"op": name + " (counts only)", "size": n, "latency_us": lat, "kernel_us": ker, "parity": ok,
                         "paper_gtx970_us": None})
    kb = concepts_kb(1_000_000, 32, 7)                        # Table 2: 10^6 individuals, 1..32 concepts
    for k in (1, 2, 4, 8, 16, 32):
        lat, ker, ok = measure(kb, ("AND", [A(i) for i in range(k)]) if k > 1 else ("AND", [A(0), ("TOP",)]), 30, True)
        rows.append({"op": f"and{k}", "size": 1_000_000, "latency_us": lat, "kernel_us": ker, "parity": ok,
                     "paper_gtx970_us": None})
    for n in [s for s in sizes if s >= 10]:                   # Tables 4 / card / 8: the two regimes
        for regime in ("unique", "single"):
            kb = abox.string_regime_kb(regime, n, seed=n)
            cases = [("exists", ("EXISTS", 0, False, A(0))), ("forall", ("FORALL", 0, False, A(0))),
                     ("min", ("MIN", 3, 0, False, A(0))), ("max", ("MAX", 3, 0, False, A(0))),
                     ("num", ("DRANGE", 0, 1.0, np.inf)),
                     ("str_equal", ("SEQUAL", 0, b"fixed string value")),
                     ("str_contain", ("SCONTAIN", 0, b"string"))]
            for name, tree in cases:
                lat, ker, ok = measure(kb, tree, 20, True)
                rows.append({"op": f"{name}_{regime}", "size": n, "latency_us": lat, "kernel_us": ker, "parity": ok,
                             "paper_gtx970_us": PAPER_GPU.get((f"{name}_{regime}", n))})
        for regime in ("unique", "single"):                    # distinct values: nothing to intern away
            kb = abox.string_regime_kb(regime, n, seed=n, distinct=True)
            for name, tree in (("str_equal", ("SEQUAL", 0, b"fixed string value0000000007")),
                               ("str_contain", ("SCONTAIN", 0, b"value00000007"))):
                lat, ker, ok = measure(kb, tree, 20, True)
                rows.append({"op": f"{name}_{regime}_distinct", "size": n, "latency_us": lat, "kernel_us": ker,
                             "parity": ok, "paper_gtx970_us": None})
    json.dump(rows, open(out_path, "w"), indent=1)
    print("| op | size | our eval_one latency us | our kernel us | parity | paper GTX 970 us |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['op']} | {r['size']} | {r['latency_us']:.1f} | {r['kernel_us']:.1f} | {r['parity']} | "
              f"{r['paper_gtx970_us'] if r['paper_gtx970_us'] is not None else ''} |")


if __name__ == "__main__":
    main()
