"""Pins of oracle/scores.py (reading Q14): hand-worked values, closed forms, brute-force top-k."""
import itertools

import numpy as np

from oracle import scores as osc


def test_hand_worked():
    # |P| = 4, |N| = 6
    c = [[4, 0, 0, 6],      # perfect: accuracy 1, F1 1
         [0, 0, 4, 6],      # empty hypothesis: accuracy 6/10, F1 0
         [4, 6, 0, 0],      # TOP: accuracy 4/10, F1 8/14
         [3, 1, 1, 5]]      # accuracy 8/10, F1 6/8
    assert list(osc.scores(c, osc.ACCURACY)) == [1.0, 0.6, 0.4, 0.8]
    assert list(osc.scores(c, osc.F1)) == [1.0, 0.0, 8 / 14, 0.75]
    assert list(osc.scores([[0, 0, 0, 0]], osc.ACCURACY)) == [0.0]      # no examples
    assert list(osc.scores([[0, 0, 0, 0]], osc.F1)) == [0.0]


def test_topk_brute_force():
    rng = np.random.default_rng(0)
    for trial in range(200):
        n = int(rng.integers(1, 9))
        s = rng.choice([0.0, 0.25, 0.5, 1.0], size=n)          # many ties
        k = int(rng.integers(1, n + 1))
        best = None
        for perm in itertools.permutations(range(n)):           # the lexicographically least valid order
            ok = all(s[perm[i]] > s[perm[i + 1]] or (s[perm[i]] == s[perm[i + 1]] and perm[i] < perm[i + 1])
                     for i in range(n - 1))
            if ok:
                best = perm
                break
        assert list(osc.topk(s, k)) == list(best[:k])
