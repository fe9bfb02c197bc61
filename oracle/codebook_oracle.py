"""Offline query-aware VQ codebook construction -- fp64 CPU ORACLE.

TEST INFRASTRUCTURE ONLY (same rule as a2ats_oracle.py): only tests/, smoke() and
bench.py's baseline legs may import it; it never imports the product path.

What it computes (PAPER.md "P:n" = line n; §4.2 Query-Aware Vector Quantization):

  1. H = E[q~^T q~], the second-moment matrix of post-PE query states (P:248,
     Eq. 10), estimated on a sample of m queries: H = (1/m) sum_i q_i^T q_i, plus the
     reading-Q27 jitter eps * (tr H / d) * I (the paper does not regularise H).
  2. The Cholesky factor H = L L^T, z = k~ L, C^z = C L (Eq. 16).
  3. k-means++ ("construct its codebook C^z using k-means++") on z: the first
     centre is z_{floor(u_0 n)}, centre j is the point at which the running sum of
     D(x)^2 -- the squared distance to the nearest centre so far -- first exceeds
     u_j * sum D^2 (inverse-CDF sampling with the given uniform draws u, reading Q28).
  4. Lloyd iterations on z (conventional VQ, Eq. 18 "equivalent to that of
     conventional vector quantization on transformed z"): assignment
     argmin_j ||z - c^z_j||^2 (lowest index on ties, Q12), centroid = mean of its
     points (an empty cluster keeps its centre, reading Q29), until no assignment
     changes or max_iters.
  5. C = C^z L^{-1} (Eq. 19).

Conventional VQ (Eq. 4) is the same procedure with H = I.  Pinned by
tests/test_oracle_codebook.py (closed forms, exact covers, fixpoint optimality,
monotone objective, the round trip of Eq. 19 and the query-aware advantage of Fig. 3 /
SPEC acceptance 5).
"""
from __future__ import annotations

import numpy as np

F64 = np.float64


def estimate_h(queries, eps: float = 0.0) -> np.ndarray:
    """H = (1/m) sum_i q_i^T q_i (+ eps * tr(H)/d * I)  -- P:248 (Eq. 10)."""
    Q = np.asarray(queries, dtype=F64)
    m, d = Q.shape
    H = np.zeros((d, d))
    for i in range(m):
        H += np.outer(Q[i], Q[i])
    H /= m
    if eps > 0:
        H += eps * (np.trace(H) / d) * np.eye(d)
    return H


def kmeanspp(z, L: int, u) -> np.ndarray:
    """k-means++ seeding with the given uniform draws u[0..L-1] in [0, 1):
    returns the indices of the L chosen points.  D^2(x) = min over chosen centres of
    ||x - c||^2; centre j = first index t with cumsum(D^2)[t] > u_j * sum(D^2)."""
    z = np.asarray(z, dtype=F64)
    n = z.shape[0]
    idx = [min(n - 1, int(np.floor(u[0] * n)))]
    d2 = np.sum((z - z[idx[0]]) ** 2, axis=1)
    for j in range(1, L):
        cs = np.cumsum(d2)
        tot = cs[-1]
        t = int(np.searchsorted(cs, u[j] * tot, side="right")) if tot > 0 else 0
        t = min(t, n - 1)
        idx.append(t)
        d2 = np.minimum(d2, np.sum((z - z[t]) ** 2, axis=1))
    return np.asarray(idx, dtype=np.int64)


def assign(z, Cz) -> np.ndarray:
    """argmin_j ||z_t - c^z_j||^2 per point (lowest j on ties), the squared distances
    evaluated by their definition (blocks of points only for speed)."""
    z = np.asarray(z, dtype=F64)
    Cz = np.asarray(Cz, dtype=F64)
    out = np.empty(z.shape[0], dtype=np.int64)
    for t0 in range(0, z.shape[0], 256):
        diff = z[t0:t0 + 256, None, :] - Cz[None, :, :]
        out[t0:t0 + 256] = np.argmin(np.sum(diff * diff, axis=2), axis=1)
    return out


def lloyd(z, Cz0, max_iters: int):
    """Lloyd iterations from the seeded centres; returns (C^z, labels, iterations run)."""
    z = np.asarray(z, dtype=F64)
    Cz = np.array(Cz0, dtype=F64)
    labels = assign(z, Cz)
    it = 0
    for it in range(1, max_iters + 1):
        for j in range(Cz.shape[0]):
            pts = z[labels == j]
            if len(pts):
                Cz[j] = pts.mean(axis=0)
        new = assign(z, Cz)
        changed = int(np.sum(new != labels))
        labels = new
        if changed == 0:
            break
    return Cz, labels, it


def train_codebook(keys, L: int, u, max_iters: int, H=None):
    """Query-aware codebook of P:364-367 (H given; H = None: conventional VQ, H = I).
    Returns dict(C, Cz, Lc, labels, iters)."""
    K = np.asarray(keys, dtype=F64)
    d = K.shape[1]
    Hm = np.eye(d) if H is None else np.asarray(H, dtype=F64)
    Lc = np.linalg.cholesky(Hm)                # lower, H = Lc Lc^T
    z = K @ Lc                                 # Eq. 16
    seeds = kmeanspp(z, L, u)
    Cz, labels, iters = lloyd(z, z[seeds], max_iters)
    C = Cz @ np.linalg.inv(Lc)                 # Eq. 19: C = C^z L^{-1}
    return dict(C=C, Cz=Cz, Lc=Lc, labels=labels, iters=iters, seeds=seeds)


def attention_mse(queries, keys, C, H=None) -> float:
    """J'(C) estimated on samples (Eq. 10 / 15): mean over (q, k) pairs of (q (k - k^)^T)^2,
    k^ = c_{f'(k; C)} with the codebook's own metric H (None: Euclidean)."""
    Q = np.asarray(queries, dtype=F64)
    K = np.asarray(keys, dtype=F64)
    C = np.asarray(C, dtype=F64)
    Hm = np.eye(K.shape[1]) if H is None else np.asarray(H, dtype=F64)
    codes = np.empty(K.shape[0], dtype=np.int64)
    for t0 in range(0, K.shape[0], 256):
        diff = K[t0:t0 + 256, None, :] - C[None, :, :]
        codes[t0:t0 + 256] = np.argmin(np.einsum("tld,de,tle->tl", diff, Hm, diff), axis=1)
    err = Q @ (K - C[codes]).T
    return float(np.mean(err ** 2))
