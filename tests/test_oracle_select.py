"""Pins for the oracle's approximate scores (Eq. 21, Eq. 6)
and top-K retrieval (readings Q8, Q10-Q12)."""
import numpy as np
import pytest

from oracle import a2ats_oracle as O


def explicit_bridge(q, b, d):
    h = d // 2
    f = np.array([1e4 ** (-2.0 * m / d) for m in range(h)])
    R = np.zeros((d, d))
    for m in range(h):                         # x R: (x_m, x_{m+h}) -> (x_m c - x_{m+h} s, x_{m+h} c + x_m s)
        c, s = np.cos(b * f[m]), np.sin(b * f[m])
        R[m, m], R[m, m + h] = c, s
        R[m + h, m], R[m + h, m + h] = -s, c
    return q @ R


def test_lossless_codebook_gives_exact_scores():
    # every key its own codeword (L = N, s_t = t): u^ = q~ k_t^T exactly (BJ pin)
    rng = np.random.default_rng(0)
    d, N = 64, 300
    K = rng.standard_normal((N, d))
    q = rng.standard_normal(d)
    qrot = O.wrope_query(q, 2048, O.inv_freq(d))
    u_hat = O.approx_scores(qrot, np.arange(N), K)
    exact = explicit_bridge(q, 2048, d) @ K.T
    np.testing.assert_allclose(u_hat, exact, rtol=0, atol=1e-11)


def test_single_codeword_constant_and_gather_equals_loop():
    rng = np.random.default_rng(1)
    C = rng.standard_normal((1, 16))
    s = O.approx_scores(rng.standard_normal(16), np.zeros(50, int), C)
    assert np.all(s == s[0])
    C = rng.standard_normal((40, 16))
    qr = rng.standard_normal(16)
    codes = rng.integers(0, 40, 200)
    loop = np.array([sum(qr[e] * C[c, e] for e in range(16)) for c in codes])
    np.testing.assert_allclose(O.approx_scores(qr, codes, C), loop, atol=1e-12)


def test_group_aggregate():
    x = np.array([[1.0, -2.0, 3.0], [0.5, 4.0, -1.0]])
    np.testing.assert_array_equal(O.group_aggregate(x, O.GROUP_MAX), [1.0, 4.0, 3.0])
    np.testing.assert_array_equal(O.group_aggregate(x, O.GROUP_SUM), [1.5, 2.0, 2.0])


@pytest.mark.parametrize("seed", range(12))
def test_three_selectors_agree_under_heavy_ties(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 120))
    agg = rng.integers(-4, 5, n).astype(float)        # few distinct levels: many exact ties
    S, cand, W = O.token_sets(n, int(rng.integers(1, 20)), int(rng.integers(0, 6)))
    for k in (0, 1, 3, len(cand) // 2, len(cand), len(cand) + 7):
        a = O.select_topk(agg, cand, k)
        np.testing.assert_array_equal(a, O.select_topk_threshold(agg, cand, k))
        np.testing.assert_array_equal(a, O.select_topk_bruteforce(agg, cand, k))
        assert len(a) == min(max(k, 0), len(cand))
        assert np.all(np.diff(a) > 0)


def test_k_covers_candidates_selects_all():
    agg = np.random.default_rng(5).standard_normal(500)
    S, cand, W = O.token_sets(500, 64, 4)
    np.testing.assert_array_equal(O.select_topk(agg, cand, 10_000), cand)
    assert O.select_topk(agg, cand, 0).size == 0


def test_tie_break_lowest_index():
    agg = np.array([0, 5, 5, 5, 5, 1, 5, 0, 0, 0], float)
    cand = np.arange(1, 8)
    np.testing.assert_array_equal(O.select_topk(agg, cand, 3), [1, 2, 3])
    np.testing.assert_array_equal(O.select_topk(agg, cand, 6), [1, 2, 3, 4, 5, 6])


def test_permutation_equivariance():
    # BJ pin: permuting candidate positions (codes and rows together) permutes the
    # selected set, on inputs whose cut falls between distinct levels
    rng = np.random.default_rng(6)
    N, L, d, G = 600, 32, 16, 4
    C = rng.standard_normal((L, d))
    qrot = rng.standard_normal((G, d))
    codes = rng.integers(0, L, N)
    S, cand, W = O.token_sets(N, 64, 4)
    agg = O.group_aggregate(O.approx_scores(qrot, codes, C))
    levels = np.sort(np.unique(agg[cand]))[::-1]
    counts = np.array([(agg[cand] == v).sum() for v in levels])
    k = int(np.cumsum(counts)[7])                      # cut exactly at a level boundary
    sel = O.select_topk(agg, cand, k)
    perm = rng.permutation(cand)                       # new position of each candidate
    codes2 = codes.copy()
    codes2[perm] = codes[cand]
    agg2 = O.group_aggregate(O.approx_scores(qrot, codes2, C))
    sel2 = O.select_topk(agg2, cand, k)
    mapping = dict(zip(cand, perm))
    np.testing.assert_array_equal(np.sort([mapping[t] for t in sel]), sel2)


def test_scale_invariance_of_ranking():
    # ranking on unscaled u^ equals ranking on u^/sqrt(d) (reading Q11)
    rng = np.random.default_rng(7)
    agg = rng.standard_normal(1000)
    S, cand, W = O.token_sets(1000, 64, 4)
    np.testing.assert_array_equal(O.select_topk(agg, cand, 60), O.select_topk(agg / np.sqrt(128), cand, 60))
