"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times, on outputs the
oracle can compute one by one (SURVEY 8(d) "Parity protocol per config").

* C4: 10^6 individuals x 10^6 refinement hypotheses, through both programs bench.py times
  (`value`: host compile, device counts; `e2e`: device compile from host arrays): all 10^6
  counts agree, a 1,200-root sample matches the oracle, 1,024 bitsets of the full-batch
  device program match the oracle.
* C3: 10^7 individuals, 1.6*10^8 assertions: the 8 fixed hypotheses, bitsets and counts.
* C5: 1.25*10^7 individuals, 10^8-edge role: the config's 10^5 cardinality/datatype-heavy
  batch through both programs, a 2,000-root oracle sample.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import setsem
from synth import abox, hyps
from synth.format import flatten

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _hedl():
    import paper_2412_00802_b200 as hedl
    hedl.lib()
    return hedl


def _c4():
    import bench

    class A:
        n_individuals, n_hyps, seed, cache = 1_000_000, 1_000_000, 4, "/tmp/hedl_cache"
    return bench.c4_inputs(A, 1)


def test_c4_full_batch_value_and_e2e_paths():
    """C4 exactly as bench.py times it (SURVEY 8(d) "C4: all counts, plus bitsets for a 1,000-
    hypothesis sample"):
      * value path: host-compiled program, counts on the device, default flags;
      * e2e path: hedl_compile_device from the rank's HOST arrays (HEDL_COMPILE_HOST_INPUT, one
        C-ABI call), device plan, counts to the host;
    all 10^6 counts of the two programs agree; 1,200 seeded roots' counts equal the oracle's;
    1,024 bitsets (four 256-root sub-ranges of the SAME full-batch device program, via
    hedl_eval_batch(first, n, want_bits)) and their counts equal the oracle's."""
    import torch
    from paper_2412_00802_b200 import dist as hdist
    hedl = _hedl()
    kb_np, nodes, kids, roots = _c4()
    n = len(roots)
    assert n == 1_000_000
    kb = hedl.hedl_kb_load(kb_np, 0)
    prog = hedl.hedl_compile(kb, nodes, kids, roots)
    counts = torch.empty((n, 4), dtype=torch.int64, device="cuda:0")
    hedl.hedl_eval_batch(kb, prog, 0, n, counts_device=True, out_counts=counts)      # bench's value path
    torch.cuda.synchronize()
    c_val = counts.cpu().numpy().view(np.uint64).copy()
    ln, lk, lr = hdist.local_arrays(nodes, kids, roots, 0, n)                          # bench's e2e inputs
    pin = [torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1)).pin_memory()
           for a in (ln, np.asarray(lk, np.uint32), np.asarray(lr, np.uint32))]
    pdev = hedl.hedl_compile_device(kb, *pin, n_nodes=len(ln), n_kids=len(lk), n_roots=len(lr))
    _, c_e2e = hedl.hedl_eval_batch(kb, pdev, 0, n)                                    # bench's e2e path
    bad = np.nonzero((c_val != c_e2e).any(axis=1))[0]
    assert len(bad) == 0, f"{len(bad)} of 10^6 roots differ between the value and e2e programs, first {bad[:5]}"
    okb = setsem.OracleKB(kb_np)
    rng = np.random.default_rng(2024)
    sample = np.sort(rng.choice(n, 1200, replace=False))
    _, oc = okb.evaluate(nodes, kids, roots[sample], want_bits=False, threads=os.cpu_count())
    bad = np.nonzero((c_val[sample] != oc).any(axis=1))[0]
    assert len(bad) == 0, f"{len(bad)} of 1200 sampled roots differ from the oracle, first {sample[bad[:5]]}"
    for first in np.sort(rng.choice(n - 256, 4, replace=False)):
        gb, gc = hedl.hedl_eval_batch(kb, pdev, int(first), 256, want_bits=True)       # same program
        rs = np.arange(first, first + 256)
        ob, oc2 = okb.evaluate(nodes, kids, roots[rs], want_bits=True, threads=os.cpu_count())
        assert np.array_equal(gc, oc2), f"counts of roots {first}..{first + 255}"
        assert np.array_equal(gb.cpu().numpy().view(np.uint32), ob), f"bitsets of roots {first}..{first + 255}"
        assert np.array_equal(gc, c_val[rs])


def test_c3_fixed_hypotheses():
    hedl = _hedl()
    kb_np = abox.c3_kb()
    trees = hyps.c3_hypotheses()
    nodes, kids, roots = flatten(trees)
    kb = hedl.hedl_kb_load(kb_np, 0)
    prog = hedl.hedl_compile(kb, nodes, kids, roots)
    gb, gc = hedl.hedl_eval_batch(kb, prog, 0, len(roots), want_bits=True)
    ob, oc = setsem.evaluate(kb_np, nodes, kids, roots, threads=os.cpu_count())
    assert np.array_equal(gc, oc)
    assert np.array_equal(gb.cpu().numpy().view(np.uint32), ob)
    for i in range(len(roots)):                    # the latency path (per-node kernels at this N)
        b1, c1 = hedl.hedl_eval_one(kb, prog, i, want_bits=True)
        assert c1 == tuple(int(v) for v in oc[i])
        assert np.array_equal(b1.cpu().numpy().view(np.uint32), ob[i])


def test_c5_full_batch_sampled():
    """C5 at its config (BASELINE configs[4]: 1.25*10^7 individuals, a 10^8-edge role + inverse,
    10^5 cardinality / datatype-heavy hypotheses) as bench.py's C5 leg runs it: the value
    program (host compile, device counts) and the e2e program (device compile from host arrays)
    agree on all 10^5 counts; a seeded 2,000-root sample equals the oracle's counts
    (tests/golden/c5_sample_expected.npz, written by tools/make_c5_expected.py from oracle/
    only -- ~2 CPU-hours -- with digests of the generated inputs), and 100 of those roots are
    re-derived by the oracle live."""
    import torch
    from paper_2412_00802_b200 import dist as hdist
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import make_c5_expected as mk
    hedl = _hedl()
    exp = np.load(os.path.join(ROOT, "tests", "golden", "c5_sample_expected.npz"))
    kb_np = abox.c5_kb()
    nodes, kids, roots = hyps.batch_arrays("c5", kb_np, mk.N_HYPS, mk.HYP_SEED)
    assert str(exp["kb_sha"]) == mk.kb_digest(kb_np), "C5 KB generator changed: regenerate the expectations"
    assert str(exp["hyps_sha"]) == mk.digest(nodes, kids, roots), "C5 batch generator changed: regenerate"
    sample = exp["sample"].astype(np.int64)
    assert np.array_equal(sample, mk.sample_roots(len(roots)))
    n = len(roots)
    kb = hedl.hedl_kb_load(kb_np, 0)
    prog = hedl.hedl_compile(kb, nodes, kids, roots)
    counts = torch.empty((n, 4), dtype=torch.int64, device="cuda:0")
    hedl.hedl_eval_batch(kb, prog, 0, n, counts_device=True, out_counts=counts)
    torch.cuda.synchronize()
    c_val = counts.cpu().numpy().view(np.uint64).copy()
    ln, lk, lr = hdist.local_arrays(nodes, kids, roots, 0, n)
    pdev = hedl.hedl_compile_device(kb, ln, lk, lr)
    _, c_e2e = hedl.hedl_eval_batch(kb, pdev, 0, n)
    bad = np.nonzero((c_val != c_e2e).any(axis=1))[0]
    assert len(bad) == 0, f"{len(bad)} of 10^5 roots differ between the value and e2e programs"
    bad = np.nonzero((c_val[sample] != exp["counts"]).any(axis=1))[0]
    assert len(bad) == 0, f"{len(bad)} of 2000 sampled roots differ from the oracle, first {sample[bad[:5]]}"
    live = sample[np.random.default_rng(7).choice(len(sample), 100, replace=False)]
    _, oc = setsem.evaluate(kb_np, nodes, kids, roots[live], want_bits=False, threads=os.cpu_count())
    assert np.array_equal(c_val[live], oc)
