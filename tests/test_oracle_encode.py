"""Pins for the oracle's query-aware VQ encoding (Eq. 14, Cholesky
form Eqs. 15-18, inference-time quantization Eq. 20)."""
import numpy as np
from scipy.spatial.distance import cdist

from oracle import a2ats_oracle as O


def spd(rng, d, cond=None):
    A = rng.standard_normal((d, d))
    H = A @ A.T / d + 0.01 * np.eye(d)
    if cond is not None:
        w, U = np.linalg.eigh(H)
        w = np.geomspace(1.0, cond, d)
        H = (U * w) @ U.T
    return 0.5 * (H + H.T)


def test_spec_worked_example(golden):
    g = golden("spec_quantize_example.json")
    k, C, H = np.array([g["k"]]), np.array(g["C"]), np.array(g["H"])
    assert O.qavq_encode(k, C, H)[0] == g["code_query_aware"]
    assert O.qavq_encode_zspace(k, C, H)[0] == g["code_query_aware"]
    assert O.qavq_encode_chform(k, C, H)[0] == g["code_query_aware"]
    assert O.qavq_encode(k, C, None)[0] == g["code_euclidean"]   # Euclidean tie -> lowest index
    D, n = O.qavq_expanded_terms(C, H)
    kHk = float(k[0] @ H @ k[0])
    np.testing.assert_allclose(kHk - 2 * (k[0] @ D.T) + n, g["quadratic_forms"])


def test_key_equal_codeword():
    rng = np.random.default_rng(0)
    C = rng.standard_normal((64, 16))
    H = spd(rng, 16)
    assert O.qavq_encode(C[7:8], C, H)[0] == 7
    assert all(O.qavq_encode(C, C, H) == np.arange(64))


def test_identity_metric_is_euclidean_nearest():
    # H = I reduces f' to the conventional quantizer f (Eq. 5) = library nearest neighbour
    rng = np.random.default_rng(1)
    C = rng.standard_normal((128, 32))
    X = rng.standard_normal((300, 32))
    ref = np.argmin(cdist(X, C, "sqeuclidean"), axis=1)
    np.testing.assert_array_equal(O.qavq_encode(X, C, None), ref)
    np.testing.assert_array_equal(O.qavq_encode(X, C, np.eye(32)), ref)


def test_three_forms_agree():
    # SPEC acceptance 3: quadratic form == z-space (Cholesky) argmin, 100%; plus the CH-form
    rng = np.random.default_rng(2)
    for cond in (None, 1e2, 1e4):
        d, L = 32, 256
        H = spd(rng, d, cond)
        C = rng.standard_normal((L, d))
        keys = C[rng.integers(0, L, 150)] + 0.3 * rng.standard_normal((150, d))
        a = O.qavq_encode(keys, C, H)
        np.testing.assert_array_equal(a, O.qavq_encode_zspace(keys, C, H))
        np.testing.assert_array_equal(a, O.qavq_encode_chform(keys, C, H))


def test_objective_identity_zspace():
    # SPEC acceptance 4 / Eq. 17: (k - c)H(k - c)^T == ||kL - cL||^2
    rng = np.random.default_rng(3)
    d = 24
    H = spd(rng, d, 1e3)
    L = np.linalg.cholesky(H)
    for _ in range(20):
        k, c = rng.standard_normal((2, d))
        q = (k - c) @ H @ (k - c)
        z = (k @ L - c @ L)
        assert abs(q - z @ z) <= 1e-9 * abs(q)


def test_metric_changes_the_code():
    # an anisotropic H picks a different codeword than Euclidean (Observation 3)
    C = np.array([[0.0, 1.0], [1.2, 0.0]])
    k = np.array([[1.0, 1.0]])
    assert O.qavq_encode(k, C, None)[0] == 0                       # 1.0 vs 1.04
    assert O.qavq_encode(k, C, np.diag([100.0, 1.0]))[0] == 1      # 100 vs 5


def test_duplicate_codewords_lowest_index():
    rng = np.random.default_rng(4)
    C = rng.standard_normal((10, 8))
    C[6] = C[2]
    H = spd(rng, 8)
    assert O.qavq_encode(C[2:3] + 1e-3, C, H)[0] == 2
    assert O.qavq_encode_chform(C[6:7], C, H)[0] == 2
