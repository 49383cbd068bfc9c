"""GPU parity of the lane-packed batch restriction path (K-SLICE) vs the oracle.

HEDL_EVAL_FORCE_SLICE packs every eligible restriction group, however small,
so the tiny and random cases exercise the OR packs, COUNT packs (bit-sliced
saturating counters), heavy-row chunks and the per-node fallback (n > 30).
"""
import numpy as np
import pytest

from synth import abox, hyps
from synth.format import COMPILE_COMPAT_PAPER_MAX, COMPILE_NO_CSE, flatten
from test_gpu_parity import assert_parity, gpu_eval

pytestmark = pytest.mark.gpu
FORCE = 4       # HEDL_EVAL_FORCE_SLICE
PER_NODE = 2    # HEDL_EVAL_PER_NODE
NO_FUSE = 8     # HEDL_EVAL_NO_FUSE
NO_RESTRICT_U = 16  # HEDL_EVAL_NO_RESTRICT_U
NO_USWEEP = 32  # HEDL_EVAL_NO_USWEEP


def test_slice_random_tiny():
    for seed in range(60):
        kb = abox.random_tiny_kb(seed)
        rng = np.random.default_rng(20_000 + seed)
        trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=4, n_max=6) for _ in range(40)]
        assert_parity(kb, trees, eflags=FORCE, tag=f"slice seed {seed}")
        if seed % 4 == 0:               # boolean fillers materialised instead of fused into the packs
            assert_parity(kb, trees, eflags=FORCE | NO_FUSE, tag=f"slice no-fuse {seed}")
        if seed % 4 == 1:               # no U rows from restrictions: booleans over them in full
            assert_parity(kb, trees, eflags=FORCE | NO_RESTRICT_U, tag=f"slice no-restrict-U {seed}")
        if seed % 4 == 2:               # U-only restrictions swept over all rows
            assert_parity(kb, trees, eflags=FORCE | NO_USWEEP, tag=f"slice no-U-sweep {seed}")
        if seed % 10 == 0:
            assert_parity(kb, trees, flags=COMPILE_COMPAT_PAPER_MAX, eflags=FORCE, tag=f"slice compat {seed}")


def test_slice_counts_boundaries():
    """n around the COUNT-pack limits: 0..33 (n <= 30 packed, larger n per-node), all predicates."""
    kb = abox.regime_kb("single", 40, seed=3, n_concepts=3, density=0.9)
    kb2 = abox.powerlaw_kb(5000, 3, 2, 12.0, 600, 0.5, 1.0, 0.05, 5)
    for k in (kb, kb2):
        trees = []
        for n in range(0, 34):
            for op in ("MIN", "MAX", "EXACT"):
                for inv in (False, True):
                    trees.append((op, n, 0, inv, ("ATOM", n % 3)))
                    trees.append((op, n, 0, inv, ("NOT", ("ATOM", (n + 1) % 3))))
        trees += [("EXISTS", 0, False, ("ATOM", 1)), ("FORALL", 0, True, ("ATOM", 2))]
        assert_parity(k, trees, eflags=FORCE, tag="boundaries")
        assert_parity(k, trees, flags=COMPILE_COMPAT_PAPER_MAX, eflags=FORCE, tag="boundaries compat")


@pytest.mark.parametrize("E", [513, 4097, 100_000])
def test_slice_heavy_single_subject(E):
    kb = abox.regime_kb("single", E, seed=E, n_concepts=4)
    T = ("TOP",)
    trees = []
    for c in range(4):
        trees += [("EXISTS", 0, False, ("ATOM", c)), ("FORALL", 0, False, ("ATOM", c)),
                  ("MIN", 17, 0, False, ("ATOM", c)), ("MAX", 30, 0, False, ("ATOM", c)),
                  ("EXACT", 0, 0, False, ("NOT", ("ATOM", c))), ("MIN", 2, 0, True, ("ATOM", c)),
                  ("MIN", E // 2, 0, False, ("ATOM", c))]
    trees += [("MIN", E, 0, False, T), ("MAX", E - 1, 0, False, T)]
    assert_parity(kb, trees, eflags=FORCE, tag=f"slice heavy {E}")


def test_slice_powerlaw_many_packs():
    """More than 256 restriction nodes per (level, direction): several packs per group."""
    kb = abox.powerlaw_kb(50_000, 40, 2, 8.0, 3_000, 0.7, 1.0, 0.01, 21)
    rng = np.random.default_rng(21)
    trees = []
    for _ in range(1500):
        r, inv = int(rng.integers(2)), bool(rng.integers(2))
        c = ("ATOM", int(rng.integers(40)))
        if rng.random() < 0.3:
            c = ("NOT", c)
        k = rng.integers(5)
        if k == 0:
            trees.append(("EXISTS", r, inv, c))
        elif k == 1:
            trees.append(("FORALL", r, inv, c))
        else:
            trees.append((["MIN", "MAX", "EXACT"][k - 2], int(rng.integers(0, 17)), r, inv, c))
    trees += [hyps.random_tree(rng, abox.kb_shape(kb), depth=4) for _ in range(300)]
    gb, gc = assert_parity(kb, trees, tag="slice powerlaw")          # default path (packs >= 8)
    nodes, kids, roots = flatten(trees)
    b2, c2, _ = gpu_eval(kb, nodes, kids, roots, eflags=PER_NODE)
    assert np.array_equal(b2, gb) and np.array_equal(c2, gc)
    b3, c3, _ = gpu_eval(kb, nodes, kids, roots, COMPILE_NO_CSE, eflags=FORCE)
    assert np.array_equal(b3, gb) and np.array_equal(c3, gc)


def test_slice_c4_shape():
    kb = abox.powerlaw_kb(300_000, 50, 2, 8.0, 10_000, 0.7, 1.0, 0.01, 4)
    arrays = hyps.batch_arrays("c4", kb, 20_000, 4, chunk=5000, workers=4)
    assert_parity(kb, arrays=arrays, tag="slice c4-shape")
    assert_parity(kb, arrays=arrays, eflags=NO_FUSE, tag="slice c4-shape, fillers materialised")
    assert_parity(kb, arrays=arrays, eflags=NO_FUSE | NO_RESTRICT_U, tag="slice c4-shape, round-1 planner")
    assert_parity(kb, arrays=arrays, eflags=NO_USWEEP, tag="slice c4-shape, no U sweeps")


def test_slice_tail_sizes():
    for n in (1, 31, 32, 33, 1023, 1024, 1025, 2049, 4000):
        kb = abox.random_tiny_kb(n, n=n, n_concepts=3, n_roles=2, n_data=0) if n <= 40 else \
            abox.powerlaw_kb(n, 3, 2, 4.0, min(n, 700), 0.0, 1.0, 0.05, n)
        rng = np.random.default_rng(n)
        trees = [hyps.random_tree(rng, abox.kb_shape(kb), depth=3, n_max=5) for _ in range(64)]
        assert_parity(kb, trees, eflags=FORCE, tag=f"slice N={n}")


def test_slice_ex_batched_heavy_examples():
    """EX packs batched several per launch, with heavy example rows (the hub is a positive example)."""
    from synth.format import kb_from_sets
    rng = np.random.default_rng(77)
    n = 6000
    concepts = [[i for i in range(n) if rng.random() < 0.4] for _ in range(12)]
    pairs = [(0, int(y)) for y in rng.choice(n, 3000, replace=False)]          # heavy hub 0
    pairs += [(1, int(y)) for y in rng.choice(n, 1500, replace=False)]         # heavy row 1
    pairs += [(int(x), int(rng.integers(n))) for x in rng.integers(2, n, 30000)]
    kb = kb_from_sets(n, concepts, [pairs], [], [0, 5, 7] + list(range(100, 160)), [1, 6] + list(range(200, 260)))
    trees = []
    for c in range(12):
        for inv in (False, True):
            for k in range(30):
                child = ("AND", [("ATOM", c), ("ATOM", (c + k) % 12)]) if k % 2 else ("OR", [("ATOM", c), ("NOT", ("ATOM", k % 12))])
                trees.append(("EXISTS", 0, inv, child) if k % 3 else ("MIN", k % 17, 0, inv, child))
    assert len(trees) > 512
    assert_parity(kb, trees, tag="ex batched heavy")


def test_slice_degree_ladder_dense():
    """Every 1,024-row tile holds light (<= 32), mid (33..128), big (129..512) and heavy rows,
    and the children are dense, so COUNT packs see counts far above 31 (overflow plane,
    4-pair mid groups, warp-per-row big rows, 2-slice OR steps) against n in 0..30."""
    from synth.format import kb_from_sets
    rng = np.random.default_rng(4242)
    n = 9000
    deg = (np.arange(n, dtype=np.int64) * 7919) % 600
    subj = np.repeat(np.arange(n), deg)
    obj = np.concatenate([rng.choice(n, int(d), replace=False) for d in deg])
    dens = (0.95, 0.5, 0.08, 0.99)
    concepts = [np.flatnonzero(rng.random(n) < p).tolist() for p in dens]
    kb = kb_from_sets(n, concepts, [list(zip(subj.tolist(), obj.tolist()))], [],
                      list(range(0, n, 7)), [x for x in range(3, n, 11) if x % 7])
    trees = []
    for c in range(4):
        for inv in (False, True):
            trees += [("EXISTS", 0, inv, ("ATOM", c)), ("FORALL", 0, inv, ("ATOM", c)),
                      ("EXISTS", 0, inv, ("NOT", ("ATOM", c))), ("FORALL", 0, inv, ("NOT", ("ATOM", c)))]
            for nn in (0, 1, 2, 15, 29, 30):
                for op in ("MIN", "MAX"):
                    trees.append((op, nn, 0, inv, ("ATOM", c)))
            trees.append(("EXACT", 30, 0, inv, ("ATOM", c)))
    assert_parity(kb, trees, eflags=FORCE, tag="degree ladder (forced packs)")
    assert_parity(kb, trees, tag="degree ladder (default)")
    # without EXACT lanes (packs of GE / LE only)
    trees2 = [t for t in trees if t[0] != "EXACT"]
    assert_parity(kb, trees2, eflags=FORCE, tag="degree ladder GE/LE only")


@pytest.mark.parametrize("cls", ["or", "count"])
def test_slice_pack_widths(cls):
    """Full-pack sweep widths at their boundaries (DESIGN.md items 23, 23b): a group of k
    restriction roots of one class, level and direction sweeps as a narrow pack (k <= 128,
    one thread per row, 16 B T records), a single pack (129..256), a pack pair (257..512,
    64 B records) or a pair plus a remainder; on a power-law KB with heavy rows (adaptive
    heavy chunks), medium rows, SELL light slices and a ragged last tile."""
    kb = abox.powerlaw_kb(50_000 + 77, 40, 2, 9.0, 3000, 0.5, 1.0, 0.02, seed=31)
    C = kb["concept_bits"].shape[0]
    A = lambda i: ("ATOM", i)
    fillers = [("AND", [A(i), A(j)]) for i in range(C) for j in range(i + 1, C)]
    fillers += [("OR", [A(i), ("NOT", A(j))]) for i in range(C) for j in range(C) if i != j]
    for k in (1, 100, 128, 129, 256, 257, 300, 512, 513):
        fs = fillers[:k]
        if cls == "or":
            trees = [("EXISTS", 0, False, f) if q % 2 == 0 else ("FORALL", 0, False, f) for q, f in enumerate(fs)]
        else:
            trees = [("MIN", 2 + q % 7, 0, False, f) if q % 2 == 0 else ("MAX", 1 + q % 5, 0, False, f)
                     for q, f in enumerate(fs)]
        assert_parity(kb, trees, eflags=FORCE, tag=f"pack width {cls} k={k}")
        assert_parity(kb, [(t[0], *t[1:3], True, *t[4:]) if t[0] in ("MIN", "MAX") else (t[0], t[1], True, t[3])
                           for t in trees], eflags=FORCE, tag=f"pack width {cls} k={k} inverse")
