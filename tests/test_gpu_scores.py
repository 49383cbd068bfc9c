"""Device scores + top-k (hedl_score_topk) vs oracle/scores.py: the float64
scores bit-exact (same formula, one correctly rounded division) and the top-k indices exact."""
import numpy as np
import pytest

from oracle import scores as osc
from oracle import setsem
from synth import abox, hyps
from synth.format import flatten
from test_gpu_parity import _hedl

pytestmark = pytest.mark.gpu


def _counts(rng, n, P=40, Nn=60, coarse=True):
    tp = rng.integers(0, P + 1, n)
    fp = rng.integers(0, Nn + 1, n)
    if coarse:                                           # many exactly tied scores
        tp = (tp // 10) * 10
        fp = (fp // 20) * 20
    return np.stack([tp, fp, P - tp, Nn - fp], 1).astype(np.int64)


@pytest.mark.parametrize("n,k", [(1, 1), (5, 5), (1000, 1), (1000, 37), (4096, 4096), (100_000, 1000),
                                 (1_000_000, 4096), (1_000_000, 0)])
def test_scores_topk_random(n, k):
    import torch
    hedl = _hedl()
    rng = np.random.default_rng(n + k)
    c = _counts(rng, n)
    cd = torch.from_numpy(c).cuda()
    for metric in (osc.ACCURACY, osc.F1):
        s, ti, ts = hedl.hedl_score_topk(cd, metric, k)
        ref = osc.scores(c, metric)
        assert np.array_equal(s.cpu().numpy(), ref)
        top = osc.topk(ref, k)
        assert np.array_equal(ti.cpu().numpy().astype(np.int64), top)
        assert np.array_equal(ts.cpu().numpy(), ref[top])


def test_scores_edge_cases():
    import torch
    hedl = _hedl()
    c = np.array([[0, 0, 0, 0], [3, 0, 0, 0], [0, 2, 0, 0], [0, 0, 0, 5]], dtype=np.int64)
    cd = torch.from_numpy(c).cuda()
    for metric in (osc.ACCURACY, osc.F1):
        s, ti, ts = hedl.hedl_score_topk(cd, metric, 4)
        ref = osc.scores(c, metric)
        assert np.array_equal(s.cpu().numpy(), ref)
        assert np.array_equal(ti.cpu().numpy().astype(np.int64), osc.topk(ref, 4))
    with pytest.raises(hedl.HedlError):
        hedl.hedl_score_topk(cd, 0, 5)                   # k > n
    with pytest.raises(hedl.HedlError):
        hedl.hedl_score_topk(cd, 7, 1)                   # unknown metric


def test_eval_then_topk_on_device():
    """The learner loop on the device: evaluate (counts stay on the GPU), score, top-k."""
    import torch
    hedl = _hedl()
    kb = abox.c2_kb()
    trees = hyps.c2_hypotheses(kb, 256)
    nodes, kids, roots = flatten(trees)
    k = hedl.hedl_kb_load(kb, 0)
    prog = hedl.hedl_compile(k, nodes, kids, roots)
    _, cd = hedl.hedl_eval_batch(k, prog, 0, len(roots), counts_device=True)
    s, ti, ts = hedl.hedl_score_topk(cd, osc.F1, 16)
    torch.cuda.synchronize()
    _, oc = setsem.evaluate(kb, nodes, kids, roots, threads=8)
    ref = osc.scores(oc.astype(np.int64), osc.F1)
    assert np.array_equal(s.cpu().numpy(), ref)
    assert np.array_equal(ti.cpu().numpy().astype(np.int64), osc.topk(ref, 16))
