"""The SURVEY 8(b) boundary calls beyond load / compile / eval, through the C ABI on the GPU:

* hedl_compile_text (SPEC.md:347-355 grammar + the 8(b) extensions): every golden fixture's
  hypotheses, as text, give the fixture's hand-worked instance sets and counts; SPEC's DSOME
  comparator forms equal the closed intervals of reading Q9; random trees printed as text and
  parsed back give the tree compiler's bitsets; syntax / name errors name the hypothesis and
  the byte offset (HEDL_ERR_PARSE).
* hedl_set_allocator: with torch's caching allocator installed (the binding's default) the KB
  and workspaces live in torch-accounted memory, and repeated evaluations allocate nothing.
* hedl_program_workspace_bytes + hedl_program_set_workspace: evaluations on a caller-provided
  block make no device allocation at all and give the library-managed results; a block that
  is too small fails with HEDL_ERR_OOM.
* hedl_compile_device with HOST arrays (HEDL_COMPILE_HOST_INPUT): one call from host arrays to
  a program, equal to the device-array and host-compiler programs.
"""
import numpy as np
import pytest

from golden_io import all_fixtures, load, load_names
from oracle import setsem
from synth import abox, hyps
from synth.format import flatten, tree_to_text
from test_gpu_parity import _hedl

pytestmark = pytest.mark.gpu


def _members(row, n):
    bits = np.unpackbits(np.asarray(row, dtype=np.uint32).view(np.uint8), bitorder="little")[:n]
    return set(np.nonzero(bits)[0].tolist())


@pytest.mark.parametrize("path", all_fixtures(), ids=lambda p: p.split("/")[-1])
def test_compile_text_golden(path):
    """Golden fixtures (each citing its SPEC / PAPER passage), compiled from their text."""
    hedl = _hedl()
    kb, cases, flags = load(path)
    names = load_names(path)
    k = hedl.hedl_kb_load(kb, 0)
    prog = hedl.hedl_compile_text(k, [c[0] for c in cases], names, flags)
    bits, counts = hedl.hedl_eval_batch(k, prog, 0, len(cases), want_bits=True)
    b = bits.cpu().numpy().view(np.uint32)
    for i, (text, _, members, cnt) in enumerate(cases):
        assert _members(b[i], kb["N"]) == members, text
        if cnt is not None:
            assert tuple(int(v) for v in counts[i]) == cnt, text


def test_compile_text_dsome_spec_forms():
    """SPEC.md:214-216 with SPEC's own DSOME syntax: >=v, ==v, <=v read as [v,+inf], [v,v],
    [-inf,v] (reading Q9) -- the same sets as the fixture's DRANGE forms."""
    hedl = _hedl()
    path = [p for p in all_fixtures() if p.endswith("numeric.kbt")][0]
    kb, _, _ = load(path)
    names = load_names(path)
    k = hedl.hedl_kb_load(kb, 0)
    texts = ["(DSOME age >= 18.0)", "(DSOME age == 17.0)", "(DSOME age == 10)", "(DSOME w <= 6.0)",
             "(AND (DSOME w >= 6.0) (DSOME w <= 29.0))", "(DSOME w >= -inf)"]
    want = [{0}, set(), {1}, {2}, {2}, {2}]       # a b s; s holds 5 and 30 (the AND is per conjunct)
    prog = hedl.hedl_compile_text(k, texts, names)
    bits, _ = hedl.hedl_eval_batch(k, prog, 0, len(texts), want_bits=True)
    b = bits.cpu().numpy().view(np.uint32)
    for i, t in enumerate(texts):
        assert _members(b[i], kb["N"]) == want[i], t


def test_compile_text_round_trip_random():
    """Random trees over every constructor -> text (default spellings c<id>, r<id>, d<id>) ->
    hedl_compile_text equals hedl_compile of the trees, and the oracle, bit for bit."""
    hedl = _hedl()
    for seed in range(30):
        kb = abox.random_tiny_kb(seed, n_strings=0)
        shape = abox.kb_shape(kb)
        rng = np.random.default_rng(seed + 500)
        trees = [hyps.random_tree(rng, shape, depth=4) for _ in range(16)]
        nm = {"concepts": [f"c{i}" for i in range(shape["C"])], "roles": [f"r{i}" for i in range(shape["R"])],
              "data": [f"d{i}" for i in range(shape["D"])]}
        texts = [tree_to_text(t, nm) for t in trees]
        k = hedl.hedl_kb_load(kb, 0)
        pt = hedl.hedl_compile_text(k, texts)                  # no name table: default spellings
        bt, ct = hedl.hedl_eval_batch(k, pt, 0, len(texts), want_bits=True)
        nodes, kids, roots = flatten(trees)
        ob, oc = setsem.evaluate(kb, nodes, kids, roots)
        assert np.array_equal(bt.cpu().numpy().view(np.uint32), ob), seed
        assert np.array_equal(ct, oc), seed


@pytest.mark.parametrize("texts,index,pos", [
    (["c0", "(AND c0 c9)"], 1, 8),                  # unknown concept (the KB has 4)
    (["(SOME r0 c1"], 0, 11),                       # missing ')': end of input
    (["(MIN -2 r0 c1)"], 0, 5),                     # negative cardinality
    (["(FOO c1)"], 0, 1),                           # unknown constructor
    (["c1 c2"], 0, 3),                              # trailing input
    (["(SSOME s0 EQUAL \"abc)"], 0, 16),            # unterminated string literal
    (["(SOME (INV q) c1)"], 0, 11),                 # unknown role
    (["TOP", "BOTTOM", "(DSOME d0 != 1.0)"], 2, 10),  # bad comparator
    (["(DRANGE d0 1.0 abc)"], 0, 15),               # malformed number
])
def test_compile_text_errors(texts, index, pos):
    hedl = _hedl()
    kb = abox.random_tiny_kb(3, n=20, n_concepts=4, n_roles=2, n_data=1, n_strings=1)
    k = hedl.hedl_kb_load(kb, 0)
    with pytest.raises(hedl.ParseError) as e:
        hedl.hedl_compile_text(k, texts)
    assert e.value.code == 5 and e.value.index == index and e.value.pos == pos, str(e.value)


def test_compile_text_semantic_errors():
    """Well-formed text with an invalid expression is the compiler's error (BAD_EXPR: NaN bound,
    reading Q10; n > 2^32-2, reading Q5)."""
    hedl = _hedl()
    k = hedl.hedl_kb_load(abox.c1_kb(), 0)
    for t in ("(DRANGE d0 nan 1.0)", "(MIN 4294967295 r0 c1)"):
        with pytest.raises(hedl.HedlError) as e:
            hedl.hedl_compile_text(k, [t])
        assert e.value.code == 4, t


def _batch(n_ind=200_000, n_hyps=6000, seed=9):
    kb = abox.powerlaw_kb(n_ind, 20, 2, 8.0, 3000, data_frac=0.7, data_vals_mean=1.0, ex_frac=0.01, seed=seed)
    nodes, kids, roots = hyps.batch_arrays("c4", kb, n_hyps, seed=3)
    return kb, nodes, kids, roots


def test_torch_allocator_no_alloc_after_warmup():
    """hedl_set_allocator with torch's caching allocator (the binding's default): the KB is in
    torch-accounted memory, and once a program is warm its evaluations allocate nothing."""
    import torch
    hedl = _hedl()
    kb, nodes, kids, roots = _batch()
    m0 = torch.cuda.memory_allocated(0)
    k = hedl.hedl_kb_load(kb, 0)
    assert torch.cuda.memory_allocated(0) - m0 >= k.info()["device_bytes"]
    prog = hedl.hedl_compile(k, nodes, kids, roots)
    n = len(roots)
    cdev = torch.empty((n, 4), dtype=torch.int64, device="cuda:0")
    _, c_ref = hedl.hedl_eval_batch(k, prog, 0, n)
    hedl.hedl_eval_batch(k, prog, 0, n, counts_device=True, out_counts=cdev)
    torch.cuda.synchronize()
    a0 = hedl.alloc_counters()
    for _ in range(3):
        _, c = hedl.hedl_eval_batch(k, prog, 0, n)
        hedl.hedl_eval_batch(k, prog, 0, n, counts_device=True, out_counts=cdev)
    torch.cuda.synchronize()
    assert hedl.alloc_counters() == a0
    assert np.array_equal(c, c_ref) and np.array_equal(cdev.cpu().numpy().view(np.uint64), c_ref)


def test_caller_workspace_never_allocates():
    """hedl_program_workspace_bytes sizes a block; with it installed (hedl_program_set_workspace)
    batch, bitset and latency calls make no device allocation -- from the first call on -- and
    return the library-managed results; a too-small block is HEDL_ERR_OOM."""
    import torch
    hedl = _hedl()
    kb, nodes, kids, roots = _batch()
    k = hedl.hedl_kb_load(kb, 0)
    ref = hedl.hedl_compile(k, nodes, kids, roots)
    n = len(roots)
    bref, cref = hedl.hedl_eval_batch(k, ref, 0, 64, want_bits=True)
    _, call_ref = hedl.hedl_eval_batch(k, ref, 0, n)
    prog = hedl.hedl_compile(k, nodes, kids, roots)
    need = max(prog.workspace_bytes(0, n), prog.workspace_bytes(0, 64, with_bits=True),
               max(prog.workspace_bytes(r, 1, True, hedl.HEDL_EVAL_PER_NODE) for r in range(0, n, 997)))
    assert need > 0
    buf = torch.empty(need, dtype=torch.uint8, device="cuda:0")
    prog.set_workspace(buf)
    hedl.hedl_eval_one(k, prog, 0)               # warms the KB-level latency table (once per KB)
    torch.cuda.synchronize()
    a0 = hedl.alloc_counters()
    _, c_all = hedl.hedl_eval_batch(k, prog, 0, n)
    b, c = hedl.hedl_eval_batch(k, prog, 0, 64, want_bits=True)
    cdev = torch.empty((n, 4), dtype=torch.int64, device="cuda:0")
    hedl.hedl_eval_batch(k, prog, 0, n, counts_device=True, out_counts=cdev)
    lat = [hedl.hedl_eval_one(k, prog, r) for r in range(0, n, 997)]
    torch.cuda.synchronize()
    assert hedl.alloc_counters() == a0, "a call on a caller workspace allocated device memory"
    assert np.array_equal(c_all, call_ref)
    assert np.array_equal(cdev.cpu().numpy().view(np.uint64), call_ref)
    assert np.array_equal(b.cpu().numpy(), bref.cpu().numpy()) and np.array_equal(c, cref)
    for r, (_, cc) in zip(range(0, n, 997), lat):
        assert cc == tuple(int(v) for v in call_ref[r])
    # too small: a clear OOM, no allocation behind the caller's back
    small = hedl.hedl_compile(k, nodes, kids, roots)
    tiny = torch.empty(64 << 10, dtype=torch.uint8, device="cuda:0")
    small.set_workspace(tiny)
    with pytest.raises(hedl.HedlError) as e:
        hedl.hedl_eval_batch(k, small, 0, n)
    assert e.value.code == 7 and "workspace" in str(e.value)
    small.set_workspace(None)                    # back to library memory
    _, c2 = hedl.hedl_eval_batch(k, small, 0, n)
    assert np.array_equal(c2, call_ref)


def test_compile_device_host_input():
    """hedl_compile_device straight from host arrays (pageable numpy and page-locked tensors):
    the same counts as the device-array path and the host compiler."""
    import torch
    hedl = _hedl()
    kb, nodes, kids, roots = _batch()
    k = hedl.hedl_kb_load(kb, 0)
    n = len(roots)
    _, c_host = hedl.hedl_eval_batch(k, hedl.hedl_compile(k, nodes, kids, roots), 0, n)
    p1 = hedl.hedl_compile_device(k, nodes, kids, roots)                        # pageable host arrays
    _, c1 = hedl.hedl_eval_batch(k, p1, 0, n)
    pin = [torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).reshape(-1)).pin_memory()
           for a in (nodes, np.asarray(kids, np.uint32), np.asarray(roots, np.uint32))]
    p2 = hedl.hedl_compile_device(k, *pin, n_nodes=len(nodes), n_kids=len(kids), n_roots=n)
    _, c2 = hedl.hedl_eval_batch(k, p2, 0, n)
    dev = [t.to("cuda:0") for t in pin]
    p3 = hedl.hedl_compile_device(k, *dev, n_nodes=len(nodes), n_kids=len(kids), n_roots=n)
    _, c3 = hedl.hedl_eval_batch(k, p3, 0, n)
    assert np.array_equal(c1, c_host) and np.array_equal(c2, c_host) and np.array_equal(c3, c_host)


def test_set_allocator_only_without_live_kbs():
    hedl = _hedl()
    k = hedl.hedl_kb_load(abox.c1_kb(), 0)
    with pytest.raises(hedl.HedlError) as e:
        hedl.use_torch_allocator(False)
    assert e.value.code == 1
    k.free()
