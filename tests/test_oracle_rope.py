"""Pins for the oracle's RoPE / WRoPE (Eq. 1, Eq. 3 P:92-103,
Eq. 11, Eq. 12).  Each check uses a formulation other
than the oracle's own (closed-form constants, complex multiplication,
explicit d x d matrices) so a wrong sign, pairing or frequency fails."""
import numpy as np
import pytest

from oracle import a2ats_oracle as O


def complex_rotate(x, pos, theta):
    """Independent formulation: pair (x_m, x_{m+d/2}) as x_m + i x_{m+d/2},
    multiplied by exp(i pos theta^(-2m/d))."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    h = d // 2
    freqs = np.array([theta ** (-2.0 * m / d) for m in range(h)])
    z = (x[..., :h] + 1j * x[..., h:]) * np.exp(1j * pos * freqs)
    return np.concatenate([z.real, z.imag], axis=-1)


def explicit_matrix(p, d, theta=1e4):
    """R_p as a d x d matrix, rows = images of the basis rows (x R_p convention)."""
    return np.stack([complex_rotate(np.eye(d)[r], p, theta) for r in range(d)])


def test_golden_closed_forms(golden):
    g = golden("rope_closed_form.json")
    for c in g["cases"]:
        y = O.rope_rotate(np.array(c["x"], float), c["pos"], O.inv_freq(c["d"], c["theta"]))
        np.testing.assert_allclose(y, c["y"], rtol=0, atol=1e-15, err_msg=c["why"])


def test_inv_freq_closed_form():
    f = O.inv_freq(128, 1e4)
    assert f[0] == 1.0
    assert abs(f[1] - 10 ** (-0.0625)) < 1e-16
    assert abs(f[-1] - 1e4 ** (-126 / 128)) < 1e-18
    with pytest.raises(ValueError):
        O.inv_freq(7)


def test_d2_angle():
    # the only d = 2 frequency is theta^0 = 1 rad / position: [1,0] at alpha -> [cos a, sin a]
    for alpha in [0, 1, 2, 3, 17, 2048]:
        y = O.rope_rotate([1.0, 0.0], alpha, O.inv_freq(2))
        np.testing.assert_allclose(y, [np.cos(alpha), np.sin(alpha)], atol=1e-15)


def test_matches_complex_formulation():
    rng = np.random.default_rng(0)
    for d in (2, 32, 64, 128):
        for pos in (0, 1, 63, 64, 2048, 131071):
            x = rng.standard_normal(d)
            np.testing.assert_allclose(O.rope_rotate(x, pos, O.inv_freq(d)),
                                       complex_rotate(x, pos, 1e4), atol=1e-12)


def test_orthogonality_and_composition():
    rng = np.random.default_rng(1)
    f = O.inv_freq(128)
    x = rng.standard_normal(128)
    np.testing.assert_array_equal(O.rope_rotate(x, 0, f), x)                     # R_0 = I
    for p in (1, 77, 4095, 100000):
        y = O.rope_rotate(x, p, f)
        assert abs(np.linalg.norm(y) - np.linalg.norm(x)) < 1e-10               # norm preserved
        np.testing.assert_allclose(O.rope_rotate(y, 33, f), O.rope_rotate(x, p + 33, f), atol=1e-10)
        np.testing.assert_allclose(O.rope_rotate(y, -p, f), x, atol=1e-10)


def test_relative_identity_eq3_explicit_matrices():
    # Eq. 3: R_i R_j^T = R_{i-j} (SPEC acceptance 1)
    rng = np.random.default_rng(2)
    for d in (32, 64, 128):
        for _ in range(6):
            i, j = rng.integers(-5000, 5000, size=2)
            dev = np.abs(explicit_matrix(i, d) @ explicit_matrix(j, d).T - explicit_matrix(i - j, d)).max()
            assert dev < 1e-10


def test_relative_identity_on_scores():
    # u_ij = (q R_i)(k R_j)^T = q R_{i-j} k^T (Eq. 3), at long-context positions
    rng = np.random.default_rng(3)
    f = O.inv_freq(128)
    q, k = rng.standard_normal((2, 128))
    for i, j in [(4095, 0), (131071, 131000), (70000, 3)]:
        lhs = O.rope_rotate(q, i, f) @ O.rope_rotate(k, j, f)
        rhs = O.rope_rotate(q, i - j, f) @ k
        assert abs(lhs - rhs) < 1e-9 * (np.linalg.norm(q) * np.linalg.norm(k))


def test_wrope_branches():
    rng = np.random.default_rng(4)
    f = O.inv_freq(64)
    q, k = rng.standard_normal((2, 64))
    w, b = 64, 2048
    i = 1000
    # i - j = w - 1 is local: exact relative rotation
    j = i - (w - 1)
    assert abs(O.wrope_score(q, k, i, j, w, b, f) - q @ explicit_matrix(w - 1, 64) @ k) < 1e-10
    # i - j = w is non-local: bridge R_b (strict "i-j < w")
    j = i - w
    assert abs(O.wrope_score(q, k, i, j, w, b, f) - q @ explicit_matrix(b, 64) @ k) < 1e-10
    # w = 1, b = 0: every off-diagonal score is the raw dot product
    for j in (0, 5, 999):
        assert abs(O.wrope_score(q, k, i, j, 1, 0, f) - q @ k) < 1e-12
    # keys bitwise unchanged (Eq. 12)
    kk = rng.standard_normal((5, 64))
    assert O.wrope_key(kk) is kk or np.array_equal(O.wrope_key(kk), kk)
    # post-PE query = q R_b
    np.testing.assert_allclose(O.wrope_query(q, b, f), q @ explicit_matrix(b, 64), atol=1e-12)


def test_wrope_equals_rope_when_window_covers_context():
    # w >= N: every causal pair is local -> u_ij = (q_i R_i)(k_j R_j)^T (standard RoPE, Eqs. 1-3)
    rng = np.random.default_rng(5)
    d, N = 32, 40
    f = O.inv_freq(d)
    Q, K = rng.standard_normal((2, N, d))
    for i in (0, 17, N - 1):
        for j in range(i + 1):
            std = (Q[i] @ explicit_matrix(i, d)) @ (K[j] @ explicit_matrix(j, d))
            assert abs(O.wrope_score(Q[i], K[j], i, j, N + 5, 2048, f) - std) < 1e-10


def test_token_sets():
    S, C, W = O.token_sets(4096, 64, 4)
    assert list(S) == [0, 1, 2, 3] and W[0] == 4032 and W[-1] == 4095 and len(W) == 64
    assert C[0] == 4 and C[-1] == 4031 and len(C) == 4096 - 68
    S, C, W = O.token_sets(50, 64, 4)          # N <= w: everything is local
    assert len(S) == 0 and len(C) == 0 and list(W) == list(range(50))
    S, C, W = O.token_sets(66, 64, 4)          # only 2 tokens outside the window: both sinks
    assert list(S) == [0, 1] and len(C) == 0
    S, C, W = O.token_sets(1, 64, 4)
    assert list(W) == [0]
    with pytest.raises(ValueError):
        O.token_sets(0, 64, 4)
