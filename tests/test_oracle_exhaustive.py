"""Exhaustive oracle pins at small word widths (CPU).

Brute force over every input of a tiny instantiation pins the disentangling
and the check independently of any hand-picked case:
  * w = 12, M = 3 (l = 4, k = 4): every triple in the admissible box and in the
    true no-overflow box round-trips for every excluded r; one step outside,
    the container overflows and the round trip fails (Eq. 8 / Eq. 11 are the
    operative conditions).
  * w = 16, M = 3: every single-word corruption of every stream is flagged
    when l = 6 (M l >= w), while the tie-mate l = 5 lets some through silently
    (SURVEY F2 / reading R5).
"""
import numpy as np
import pytest


def test_T7_bruteforce_box_w12(O):
    cfg = O.config_for(3, 12)
    assert (cfg.l, cfg.k) == (4, 4)
    hi = O.dynamic_range(cfg)
    assert hi == 2 ** 7 - 2 ** 4 == 112          # Eq. 11 at l = k = 4
    fails, n = O.selftest_roundtrip_box(cfg, hi)
    assert n == (2 * hi + 1) ** 3 * 3 and fails == 0


def test_T7_true_limit_and_overflow_corner_w12(O):
    """The true limit: entangled |c|(2^l+1) <= 2^(w-1)-1  ->  |c| <= 2047 // 17 = 120.
    All of [-120,120]^3 round-trips; the corner (121,121,121) overflows 12 bits."""
    cfg = O.config_for(3, 12)
    lim = (2 ** 11 - 1) // (2 ** 4 + 1)
    assert lim == 120
    fails, _ = O.selftest_roundtrip_box(cfg, lim)
    assert fails == 0
    c = np.full((3, 1), lim + 1)
    eps = O.entangle(cfg, c)
    assert (eps != c * (2 ** 4 + 1)).any()                 # wrapped in the 12-bit container
    d, flag = O.disentangle_one(cfg, eps[:, 0], 0)
    assert d.tolist() != [lim + 1] * 3


@pytest.mark.parametrize("c", [[0, 0, 0], [448, 448, 448], [-448, 448, -448], [5, -7, 100],
                               [447, -1, 0], [-448, -448, -448]])
def test_T10_every_word_corruption_flagged_w16(O, c):
    cfg = O.config_for(3, 16)
    assert (cfg.l, cfg.k) == (6, 4) and O.dynamic_range(cfg) == 448
    tried, missed, silent = O.selftest_word_sweep(cfg, c)
    assert tried == 3 * (2 ** 16 - 1)
    assert missed == 0 and silent == 0


def test_T10_tiebreak_regression_l5_w16(O):
    """The tie-mate (l, k) = (5, 5) has M l = 15 < 16: some single-word
    corruptions pass the check with wrong outputs — why R5 picks the larger l."""
    cfg = O.make_config(3, 16, 5, 5)
    total_silent = 0
    for c in ([5, -7, 100], [0, 0, 0], [100, 200, -300], [-480, 480, 0]):
        _, _, silent = O.selftest_word_sweep(cfg, c)
        total_silent += silent
    assert total_silent > 0
