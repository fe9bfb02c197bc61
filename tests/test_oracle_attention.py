"""Pins for the oracle's attention (Eq. 2 P:83-90 with WRoPE logits Eq. 11
P:283-297) and the whole decode step (P:384-397 stages 2-3), plus the
byte accounting."""
import numpy as np
from scipy.special import softmax

from oracle import a2ats_oracle as O


def rot_matrix(p, d, theta=1e4):
    h = d // 2
    R = np.zeros((d, d))
    for m in range(h):
        a = p * theta ** (-2.0 * m / d)
        c, s = np.cos(a), np.sin(a)
        R[m, m], R[m, m + h], R[m + h, m], R[m + h, m + h] = c, s, -s, c
    return R


def dense_wrope_attention(q, K, V, N, w, b):
    """Brute force Eq. 2 over all N tokens with Eq. 11 logits via explicit matrices."""
    d = q.shape[0]
    i = N - 1
    u = np.array([q @ rot_matrix(i - j if i - j < w else b, d) @ K[j] for j in range(N)])
    return softmax(u / np.sqrt(d)) @ V[:N]


def test_single_token_and_equal_logits():
    rng = np.random.default_rng(0)
    V = rng.standard_normal((1, 8))
    np.testing.assert_allclose(O.softmax_attention([3.7], V), V[0], atol=1e-15)
    V = rng.standard_normal((9, 8))
    np.testing.assert_allclose(O.softmax_attention(np.full(9, -2.5), V), V.mean(0), atol=1e-14)


def test_full_selection_equals_dense_bruteforce():
    # K >= |Cand| => selective attention == dense WRoPE attention (BJ "results match brute force when K = N")
    rng = np.random.default_rng(1)
    d, N, L, G = 32, 150, 16, 2
    C = rng.standard_normal((L, d))
    codes = rng.integers(0, L, N)
    K = C[codes] + 0.1 * rng.standard_normal((N, d))
    V = rng.standard_normal((N, d))
    q = rng.standard_normal((G, d))
    r = O.decode_step_pair(q, K, V, codes, C, N, window=16, bridge=2048, n_sink=4, topk=N)
    for g in range(G):
        np.testing.assert_allclose(r["out"][g], dense_wrope_attention(q[g], K, V, N, 16, 2048), atol=1e-12)
    assert len(r["sel_rows"]) == N


def test_window_covering_context_is_standard_rope_attention():
    # w >= N: WRoPE == standard RoPE attention with q_i R_i and k_j R_j (BJ pin)
    rng = np.random.default_rng(2)
    d, N = 16, 40
    K, V = rng.standard_normal((2, N, d))
    q = rng.standard_normal(d)
    i = N - 1
    u = np.array([(q @ rot_matrix(i, d)) @ (K[j] @ rot_matrix(j, d)) for j in range(N)])
    ref = softmax(u / np.sqrt(d)) @ V
    r = O.decode_step_pair(q[None], K, V, np.zeros(N, int), np.zeros((1, d)), N,
                           window=N + 3, bridge=2048, n_sink=4, topk=5)
    np.testing.assert_allclose(r["out"][0], ref, atol=1e-12)


def test_unselected_mass_bound():
    # ||o_sel - o_exact|| <= 2 max||v|| * (softmax mass of unselected tokens)
    rng = np.random.default_rng(3)
    d, N, L = 32, 400, 64
    C = rng.standard_normal((L, d))
    codes = rng.integers(0, L, N)
    K = C[codes] + 0.1 * rng.standard_normal((N, d))
    V = rng.standard_normal((N, d))
    q = 2.0 * rng.standard_normal((1, d))
    w, b = 64, 2048
    r = O.decode_step_pair(q, K, V, codes, C, N, window=w, bridge=b, n_sink=4, topk=40)
    exact = dense_wrope_attention(q[0], K, V, N, w, b)
    i = N - 1
    u = np.array([q[0] @ rot_matrix(i - j if i - j < w else b, d) @ K[j] for j in range(N)])
    p = softmax(u / np.sqrt(d))
    unselected = np.setdiff1d(np.arange(N), r["sel_rows"])
    bound = 2 * np.linalg.norm(V, axis=1).max() * p[unselected].sum()
    assert np.linalg.norm(r["out"][0] - exact) <= bound + 1e-12


def test_decode_step_structure():
    rng = np.random.default_rng(4)
    B, Hq, Hkv, d, N, L = 2, 4, 2, 16, 200, 8
    C = rng.standard_normal((Hkv, L, d))
    codes = rng.integers(0, L, (B, Hkv, N))
    K, V = rng.standard_normal((2, B, Hkv, N, d))
    q = rng.standard_normal((B, Hq, d))
    out, sel = O.decode_step(q, K, V, codes, C, N, window=64, bridge=2048, n_sink=4, topk=20)
    assert out.shape == (B, Hq, d) and sel.shape == (B, Hkv, 20)
    assert np.all(sel >= 4) and np.all(sel < N - 64)
    # selected tokens all score at least as high as any unselected candidate
    for b in range(B):
        for h in range(Hkv):
            r = O.decode_step_pair(q[b, 2 * h:2 * h + 2], K[b, h], V[b, h], codes[b, h], C[h], N, topk=20)
            S, cand, W = O.token_sets(N, 64, 4)
            rest = np.setdiff1d(cand, r["sel"])
            assert r["agg"][r["sel"]].min() >= r["agg"][rest].max()
            np.testing.assert_array_equal(r["sel"], sel[b, h])


def test_accounting(golden):
    g = golden("paper_constants.json")
    assert O.aux_mem_ratio(128, 2, 2) == 0.0078125
    assert round(O.aux_mem_ratio(128, 2, 2), 3) == g["aux_mem_table1"]
    assert O.aux_mem_ratio(64, 2, 2) == 0.015625
    # |Sel| = K + 68 at K = ceil(0.06 N): sparsity ~0.06 as in Table 1
    from synth import budget_k
    for n in (32768, 65536, 131072):
        s = O.sparsity_ratio(budget_k(n) + g["n_sink"] + g["recent"], n)
        assert abs(s - g["sparsity_table1_llama"]) < 0.003
    assert O.sparsity_ratio(1000, 1000) == 1.0
