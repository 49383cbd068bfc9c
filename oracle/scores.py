"""Hypothesis scores and top-k selection -- TEST INFRASTRUCTURE ONLY (the oracle side of the
device scoring of SURVEY 8(f) NEXT-3).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline may import this package.

Reading Q14: the paper reports covered positives / negatives only;
the scores are the learner's usual ones, in float64:
  accuracy = (TP + TN) / (|P| + |N|)        (0 when there are no examples)
  F1       = 2 TP / (2 TP + FP + FN)        (0 when the denominator is 0)
with |P| = TP + FN and |N| = FP + TN (Alg. 15).  top-k = the k highest
scores, ties broken by the lower hypothesis index.
"""
import numpy as np

ACCURACY, F1 = 0, 1


def scores(counts, metric: int) -> np.ndarray:
    c = np.asarray(counts, dtype=np.float64).reshape(-1, 4)
    tp, fp, fn, tn = c[:, 0], c[:, 1], c[:, 2], c[:, 3]
    if metric == ACCURACY:
        num, den = tp + tn, tp + fp + fn + tn
    elif metric == F1:
        num, den = 2.0 * tp, 2.0 * tp + fp + fn
    else:
        raise ValueError(metric)
    out = np.zeros(len(c), dtype=np.float64)
    nz = den > 0
    out[nz] = num[nz] / den[nz]
    return out


def topk(s, k: int) -> np.ndarray:
    """Indices of the k largest scores, descending, ties by ascending index (a full stable sort)."""
    s = np.asarray(s, dtype=np.float64)
    order = np.lexsort((np.arange(len(s)), -s))
    return order[:k]
