"""Pins of the offline codebook oracle (oracle/codebook_oracle.py) against
closed forms, exact covers, optimality conditions and the paper's claim -- nothing here
re-types the oracle's own formulas."""
import numpy as np
import pytest

from oracle import codebook_oracle as CB


def test_h_estimate_closed_forms():
    m, d = 6, 6
    Q = np.sqrt(m) * np.eye(d)                            # rows of sqrt(m) I -> H = I exactly
    np.testing.assert_allclose(CB.estimate_h(Q), np.eye(d), rtol=0, atol=1e-15)
    q = np.array([[1.0, 2.0, -3.0]])                      # one query: rank one, H q^T = |q|^2 q^T
    H = CB.estimate_h(q)
    assert np.linalg.matrix_rank(H) == 1
    np.testing.assert_allclose(H @ q[0], 14.0 * q[0])
    rng = np.random.default_rng(0)                        # empirical moments of N(0, diag(1, 4))
    Z = rng.standard_normal((100000, 2)) * np.array([1.0, 2.0])
    np.testing.assert_allclose(np.diag(CB.estimate_h(Z)), [1.0, 4.0], rtol=0.05)
    He = CB.estimate_h(q, eps=0.5)                        # jitter eps * tr(H)/d * I makes it SPD
    np.testing.assert_allclose(He - H, 0.5 * 14.0 / 3 * np.eye(3))
    np.linalg.cholesky(He)


def test_kmeanspp_inverse_cdf_by_hand():
    z = np.array([[0.0, 0.0], [1.0, 0.0], [3.0, 0.0]])    # D^2 from point 0: 0, 1, 9 (sum 10)
    assert list(CB.kmeanspp(z, 2, [0.0, 0.5])) == [0, 2]  # cumsum 0, 1, 10 > 5 first at index 2
    assert list(CB.kmeanspp(z, 2, [0.0, 0.05])) == [0, 1]  # > 0.5 first at index 1
    assert list(CB.kmeanspp(z, 2, [0.7, 0.0])) == [2, 0]  # first centre floor(0.7 * 3) = 2; D^2 9,4,0
    # an already chosen point (D^2 = 0) is never chosen again while others are left
    assert sorted(CB.kmeanspp(z, 3, [0.0, 0.99, 0.0])) == [0, 1, 2]


def test_exact_cover_gives_zero_error():
    rng = np.random.default_rng(1)
    K = rng.standard_normal((64, 8))
    r = CB.train_codebook(K, 64, rng.random(64), 10)
    assert sorted(r["seeds"]) == list(range(64))          # every point chosen once
    np.testing.assert_allclose(r["C"][r["labels"]], K, atol=1e-12)


def test_two_separated_clusters_recover_means():
    rng = np.random.default_rng(2)
    a = rng.standard_normal((500, 4)) * 0.1 + np.array([5.0, 0, 0, 0])
    b = rng.standard_normal((500, 4)) * 0.1 - np.array([5.0, 0, 0, 0])
    K = np.concatenate([a, b])
    r = CB.train_codebook(K, 2, rng.random(2), 20)
    got = r["C"][np.argsort(r["C"][:, 0])]
    np.testing.assert_allclose(got, [b.mean(0), a.mean(0)], atol=1e-9)   # closed-form cluster means


def _aniso(seed, d, cond=100.0):
    rng = np.random.default_rng(seed)
    A = np.linalg.qr(rng.standard_normal((d, d)))[0] * np.sqrt(np.logspace(0, np.log10(cond), d))
    return rng, A


def test_lloyd_fixpoint_and_monotone_objective():
    rng, A = _aniso(3, 8)
    K = rng.standard_normal((600, 8))
    H = A @ A.T
    Lc = np.linalg.cholesky(H)
    z = K @ Lc
    seeds = CB.kmeanspp(z, 12, rng.random(12))
    J = []
    for it in range(1, 8):                                # objective after 1, 2, ... iterations
        Cz, labels, _ = CB.lloyd(z, z[seeds], it)
        J.append(np.mean(np.sum((z - Cz[labels]) ** 2, axis=1)))
    assert all(b <= a + 1e-12 for a, b in zip(J, J[1:]))
    Cz, labels, iters = CB.lloyd(z, z[seeds], 200)
    assert iters < 200
    d2 = ((z[:, None, :] - Cz[None]) ** 2).sum(2)        # brute-force optimality of the fixpoint
    np.testing.assert_array_equal(labels, np.argmin(d2, axis=1))
    for j in range(12):
        if np.any(labels == j):
            np.testing.assert_allclose(Cz[j], z[labels == j].mean(0), atol=1e-12)
    # objective identity (Eq. 18) and the round trip of Eq. 19
    C = Cz @ np.linalg.inv(Lc)
    np.testing.assert_allclose(C @ Lc, Cz, atol=1e-9)
    jq = np.mean([(K[t] - C[labels[t]]) @ H @ (K[t] - C[labels[t]]) for t in range(len(K))])
    np.testing.assert_allclose(jq, J[-1] if iters <= 7 else np.mean(np.sum((z - Cz[labels]) ** 2, 1)), rtol=1e-9)


def test_query_aware_advantage_over_seeds():
    """SPEC acceptance 5 / the paper's Fig. 3 claim: over 20 seeds of anisotropic
    synthetic data (cond(H) = 100, L = 64, n = 4096, d = 32), the query-aware codebook has the
    lower mean attention-score MSE, and wins in at least 15 of the 20 seeds."""
    wins, qa_all, cv_all = 0, [], []
    for seed in range(20):
        rng, A = _aniso(100 + seed, 32)
        Qtrain = rng.standard_normal((4096, 32)) @ A.T    # post-PE queries, E[q^T q] = A A^T
        K = rng.standard_normal((4096, 32))
        H = CB.estimate_h(Qtrain)
        u = rng.random(64)
        qa = CB.train_codebook(K, 64, u, 25, H=H)
        cv = CB.train_codebook(K, 64, u, 25, H=None)
        Qtest = rng.standard_normal((512, 32)) @ A.T
        e_qa = CB.attention_mse(Qtest, K, qa["C"], H)
        e_cv = CB.attention_mse(Qtest, K, cv["C"], None)
        qa_all.append(e_qa)
        cv_all.append(e_cv)
        wins += e_qa < e_cv
    assert np.mean(qa_all) < np.mean(cv_all)
    assert wins >= 15, wins
