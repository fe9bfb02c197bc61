"""GPU parity of the offline codebook construction (a2ats_qavq_train) against
the fp64 oracle (oracle/codebook_oracle.py) on the same inputs (bf16 keys / queries, the
same k-means++ draws u): H within 1e-12, the Lloyd assignment of every key identical (integer
decisions), iterations identical, the codebook within 1e-9; plus the query-aware advantage
measured on GPU-built codebooks."""
import numpy as np
import pytest
import torch

from oracle import codebook_oracle as CB

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2502_12665_b200 import binding as Bd


def _data(seed, n, m, d, cond=100.0, clusters=0):
    g = torch.Generator().manual_seed(seed)
    A = torch.linalg.qr(torch.randn((d, d), generator=g, dtype=torch.float64))[0] * torch.sqrt(
        torch.logspace(0, np.log10(cond), d, dtype=torch.float64))
    Q = (torch.randn((m, d), generator=g, dtype=torch.float64) @ A.T).to(torch.bfloat16)
    if clusters:
        cent = torch.randn((clusters, d), generator=g, dtype=torch.float64) * 3
        K = cent[torch.randint(0, clusters, (n,), generator=g)] + torch.randn((n, d), generator=g, dtype=torch.float64)
    else:
        K = torch.randn((n, d), generator=g, dtype=torch.float64)
    return K.to(torch.bfloat16), Q, torch.rand((n,), generator=g, dtype=torch.float64), A


def gpu_train(K, L, u, iters, Q=None, eps=0.0):
    n, d = K.shape
    C = torch.empty((L, d), dtype=torch.float64, device="cuda")
    H = torch.empty((d, d), dtype=torch.float64, device="cuda")
    lab = torch.empty((n,), dtype=torch.int32, device="cuda")
    info = torch.zeros((2,), dtype=torch.int32, device="cuda")
    Bd.a2ats_qavq_train(K.cuda(), L, u[:L].cuda(), iters, queries=None if Q is None else Q.cuda(), eps=eps,
                        C_out=C, H_out=H, labels_out=lab, info_out=info)
    torch.cuda.synchronize()
    return C.cpu().numpy(), H.cpu().numpy(), lab.cpu().numpy(), info.cpu().numpy()


@pytest.mark.parametrize("n,m,d,L,clusters,query_aware", [(2048, 2048, 32, 64, 0, True), (3000, 1500, 128, 256, 40, True),
                                                           (4096, 0, 64, 100, 0, False), (1000, 500, 16, 7, 3, True)])
def test_train_matches_oracle(n, m, d, L, clusters, query_aware):
    K, Q, u, _ = _data(n + d + L, n, max(m, 1), d, clusters=clusters)
    eps = 1e-6 if query_aware else 0.0
    C, H, lab, info = gpu_train(K, L, u, 40, Q if query_aware else None, eps=eps)
    assert info[1] == 0
    Kn = K.double().numpy()
    Href = CB.estimate_h(Q.double().numpy(), eps) if query_aware else None
    if query_aware:
        np.testing.assert_allclose(H, Href, rtol=1e-12, atol=1e-12 * np.abs(Href).max())
    ref = CB.train_codebook(Kn, L, u[:L].numpy(), 40, H=Href)
    np.testing.assert_array_equal(lab, ref["labels"])            # every Lloyd decision identical
    assert info[0] == ref["iters"]
    np.testing.assert_allclose(C, ref["C"], rtol=0, atol=1e-9 * np.abs(ref["C"]).max())


def test_exact_cover_and_conventional_identity():
    K, Q, u, _ = _data(9, 256, 16, 32)
    C, H, lab, info = gpu_train(K, 256, u, 10)                  # L = n: every key its own codeword
    np.testing.assert_allclose(H, np.eye(32))
    np.testing.assert_array_equal(C[lab], K.double().numpy())


def test_query_aware_advantage_gpu():
    """The Fig. 3 claim on codebooks built by the GPU: over 8 seeds the query-aware
    codebook has the lower attention-score MSE on fresh queries in every mean and >= 6 seeds."""
    wins, qa, cv = 0, [], []
    for seed in range(8):
        K, Q, u, A = _data(300 + seed, 4096, 4096, 32)
        Cq, Hq, _, _ = gpu_train(K, 64, u, 25, Q)
        Cc, _, _, _ = gpu_train(K, 64, u, 25, None)
        g = torch.Generator().manual_seed(900 + seed)          # fresh queries of the same law
        Qt = (torch.randn((512, 32), generator=g, dtype=torch.float64) @ A.T).numpy()
        eq = CB.attention_mse(Qt, K.double().numpy(), Cq, Hq)
        ec = CB.attention_mse(Qt, K.double().numpy(), Cc, None)
        qa.append(eq)
        cv.append(ec)
        wins += eq < ec
    assert np.mean(qa) < np.mean(cv) and wins >= 6, (qa, cv)
