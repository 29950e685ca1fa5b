"""Pins of the oracle's prose-search MSTopK (SURVEY F3 TK_SEARCH_PROSE, reading Q33),
against a trial sequence worked by hand, the exact top-k of Eq. 2 it must converge to, and the
invariants of the two-threshold selection (Alg. 1 l.25-29) at every N."""
import numpy as np
import pytest

import gradgen
import oracle
from oracle import RAND_FIRST


def test_hand_worked_bracket_then_bisect():
    # a = 1..8, a-bar = 4.5, k = 2.  Trials (worked by hand from P:148):
    #  t=4.5  : {5,6,7,8}  nnz 4 > 2  -> double          (k2 = 4, thres2 = 4.5)
    #  t=9    : {}         nnz 0 <= 2 -> bracket [4.5, 9] (k1 stays 0: not > 0)
    #  t=6.75 : {7,8}      nnz 2 <= 2 -> k1 = 2, thres1 = 6.75; bracket [4.5, 6.75]
    #  t=5.625: {6,7,8}    nnz 3 > 2  -> k2 = 3, thres2 = 5.625
    x = np.array([1, -2, 3, 4, -5, 6, 7, -8], np.float32)
    res = oracle.mstopk_prose(x, 2, 4, rand_mode=RAND_FIRST)
    assert [t[1] for t in res.trials] == [4.5, 9.0, 6.75, 5.625]
    assert [t[3] for t in res.trials] == [4, 0, 2, 3]
    assert (res.k1, res.thres1, res.k2, res.thres2) == (2, 6.75, 3, 5.625)
    assert res.idx.tolist() == [6, 7] and res.val.tolist() == [7.0, -8.0]


def test_hand_worked_halving():
    # one large element: a = (100, 1, 1, 1), a-bar = 25.75, k = 3.  t = 25.75: nnz 1 < 3 -> halve
    # 12.875 (1) -> 6.4375 (1) -> 3.21875 (1) -> 1.609375 (1) -> 0.8046875 (4 > 3): bracket
    x = np.array([100, 1, -1, 1], np.float32)
    res = oracle.mstopk_prose(x, 3, 6, rand_mode=RAND_FIRST)
    assert [t[1] for t in res.trials] == [25.75, 12.875, 6.4375, 3.21875, 1.609375, 0.8046875]
    assert (res.k1, res.k2) == (1, 4)
    # window of the first k - k1 = 2 of iota2 = {1, 2, 3}
    assert res.idx.tolist() == [0, 1, 2]


@pytest.mark.parametrize("dist", ["G", "L"])
@pytest.mark.parametrize("d,k", [(1000, 10), (4097, 1), (65537, 655)])
def test_converges_to_exact_topk_when_the_kth_is_untied(dist, d, k):
    x = gradgen.gradient(d, dist, cfg=501)
    s = np.sort(np.abs(x))[::-1]
    assert s[k - 1] > s[k]  # the k-th largest magnitude is not tied with the (k+1)-th
    res = oracle.mstopk_prose(x, k, 52)
    idx, val = oracle.exact_topk(x, k)
    assert res.k1 == k
    assert np.array_equal(res.idx, idx) and np.array_equal(res.val.view(np.uint32), val.view(np.uint32))


@pytest.mark.parametrize("N", [1, 2, 3, 5, 10, 30])
@pytest.mark.parametrize("dist", ["G", "L", "ties8", "H"])
def test_selection_invariants(N, dist):
    d, k = 20001, 137
    x = gradgen.gradient(d, dist, cfg=502)
    a = np.abs(x).astype(np.float64)
    res = oracle.mstopk_prose(x, k, N, seed=5)
    assert len(res.idx) == k and np.all(np.diff(res.idx.astype(np.int64)) > 0)
    assert res.k1 <= k <= res.k2
    sel = a[res.idx.astype(np.int64)]
    # every element at or above thres1 is selected; every selected one is >= thres2
    if res.k1:
        assert np.count_nonzero(a >= res.thres1) == res.k1
        assert np.all(np.isin(np.nonzero(a >= res.thres1)[0], res.idx))
    assert np.all(sel >= res.thres2)
    # no trial count is inconsistent with a fresh count at its threshold
    for _, t, _, nnz in res.trials:
        assert nnz == np.count_nonzero(a >= t)


def test_all_zero_and_k_equals_d():
    z = np.zeros(64, np.float32)
    res = oracle.mstopk_prose(z, 5, 10, rand_mode=RAND_FIRST)
    assert res.idx.tolist() == [0, 1, 2, 3, 4]
    x = gradgen.gradient(100, "G", cfg=503)
    assert oracle.mstopk_prose(x, 100, 3).idx.tolist() == list(range(100))


def test_compress_selector_prose():
    g = gradgen.gradient(5000, "G", cfg=504)
    r = gradgen.gradient(5000, "G", cfg=505) * np.float32(0.1)
    c = oracle.compress(g, r, 50, 10, selector="prose", seed=1)
    acc = (g + r).astype(np.float32)
    assert np.array_equal(c.sel.idx, oracle.mstopk_prose(acc, 50, 10, seed=1).idx)
    assert np.all(c.residual[c.sel.idx.astype(np.int64)] == 0)
