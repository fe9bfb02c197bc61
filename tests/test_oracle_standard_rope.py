"""Pins for the oracle's standard-RoPE step (the ablation "Baseline" / "QAVQ" configurations,
PAPER.md P:419-427), each against something other than the function itself: post-PE keys built
with explicit d x d rotation matrices (complex-multiplication formulation), the WRoPE oracle with
a window covering the context (which equals standard RoPE attention, the BJ pin already pinned),
and exact logits from a lossless codebook."""
import numpy as np

from oracle import a2ats_oracle as O
from test_oracle_rope import explicit_matrix


def _post_pe(keys, d=16):
    return np.stack([keys[j] @ explicit_matrix(j, d) for j in range(keys.shape[0])])


def test_all_rows_selected_equals_wrope_with_full_window():
    """Every candidate selected (topk >= |Cand|): standard-RoPE attention over post-PE keys ==
    the WRoPE oracle on pre-PE keys with w >= N (Eq. 11 then rotates every row by R_{i-j})."""
    rng = np.random.default_rng(3)
    d, n, G = 16, 40, 2
    q = rng.standard_normal((G, d))
    k = rng.standard_normal((n, d))
    v = rng.standard_normal((n, d))
    C = rng.standard_normal((8, d))
    codes = rng.integers(0, 8, n)
    std = O.decode_step_pair_standard(q, _post_pe(k, d), v, codes, C, n, window=5, n_sink=2, topk=1000,
                                      freqs=O.inv_freq(d))
    ref = O.decode_step_pair(q, k, v, codes, C, n, window=n + 1, bridge=7, n_sink=2, topk=1000, freqs=O.inv_freq(d))
    assert np.array_equal(np.sort(std["sel_rows"]), np.arange(n))
    np.testing.assert_allclose(std["out"], ref["out"], rtol=1e-12, atol=1e-12)


def test_lossless_codebook_scores_are_exact_standard_logits():
    """Codebook = the post-PE keys, code t = t: approximate score = exact (q R_i) . (k_t R_t),
    with both rotations as explicit matrices."""
    rng = np.random.default_rng(4)
    d, n = 16, 30
    q = rng.standard_normal((1, d))
    k = rng.standard_normal((n, d))
    kp = _post_pe(k, d)
    r = O.decode_step_pair_standard(q, kp, rng.standard_normal((n, d)), np.arange(n), kp, n, window=4,
                                    n_sink=1, topk=5, freqs=O.inv_freq(d))
    exact = (q[0] @ explicit_matrix(n - 1, d)) @ kp.T
    np.testing.assert_allclose(r["scores"][0], exact, rtol=1e-12, atol=1e-12)
    # the top-K are the 5 largest exact logits among the candidates [1, n - 4)
    cand = np.arange(1, n - 4)
    np.testing.assert_array_equal(r["sel"], np.sort(cand[np.argsort(-exact[cand], kind="stable")[:5]]))


def test_relative_position_invariance():
    """Standard RoPE attention depends on i - j only: shifting every position by s (keys
    re-rotated at j + s, query at i + s) leaves the output unchanged (Eq. 3)."""
    rng = np.random.default_rng(5)
    d, n, s = 16, 24, 9
    q = rng.standard_normal((1, d))
    k = rng.standard_normal((n + s, d))
    v = rng.standard_normal((n + s, d))
    kp = _post_pe(k, d)
    # context of n tokens, and the same tokens placed at positions s .. s + n - 1 behind s pad tokens
    a = O.decode_step_pair_standard(q, kp[:n], v[:n], np.zeros(n, int), np.zeros((1, d)), n, window=n + 1,
                                    n_sink=0, topk=0, freqs=O.inv_freq(d))
    ks = np.concatenate([np.zeros((s, d)), np.stack([k[j] @ explicit_matrix(j + s, d) for j in range(n)])])
    vs = np.concatenate([np.zeros((s, d)), v[:n]])
    b = O.decode_step_pair_standard(q, ks, vs, np.zeros(n + s, int), np.zeros((1, d)), n + s, window=n,
                                    n_sink=0, topk=0, freqs=O.inv_freq(d))
    np.testing.assert_allclose(a["out"], b["out"], rtol=1e-12, atol=1e-12)
