"""A^2ATS decode-time retrieval path -- fp64 CPU ORACLE.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call
or execute anything under ``oracle/``.  The product path
(``paper_2502_12665_b200``) never imports it, and this module never imports
the product path: the two share no code, tables or constants.

What it computes (PAPER.md = arXiv 2502.12665 LaTeX source; "P:n" = line n):

  1. RoPE rotation R_p (Eq. 1) and its relative identity (Eq. 3,
     P:92-103).  Readings Q1-Q4 of DESIGN.md fix theta = 1e4, the half-split
     pairing (m, m + d/2), the sign convention of HF ``rotate_half`` and 0-based
     positions.
  2. Windowed RoPE (Eq. 11 ``eq:wrope``) and its post-PE states
     q~ = q R_b, k~ = k (Eq. 12).
  3. Query-aware VQ encoding f'(k; C) = argmin_j (k - c_j) H (k - c_j)^T
     (Eq. 14), the Cholesky/z-space form (Eqs. 15-18)
     and the expanded "CH-form" argmin_j (c_j H c_j^T - 2 k H c_j^T).
  4. The approximate score u^_{i,j} = q~_i c_{s_j} (Eq. 21; also
     Eq. 6), aggregated over a GQA group (reading Q10: max).
  5. Top-K retrieval over the candidates with the static
     4 sinks + 64-token window; ties by lowest token index (Q12);
     disjoint budget semantics (Q8).  Two independent implementations
     (sort-based and count-weighted level threshold).
  6. Exact softmax attention over Sel = Sinks u TopK u Window (Eq. 2,
     P:83-90) with WRoPE logits (Eq. 11): bridge rotation for non-local
     tokens, exact relative rotation inside the window.

Everything is scalar-definition numpy in float64; inputs given as bf16/fp32
are converted exactly to float64 by the caller.  No blocking, fusion or
reordering beyond what the paper's definitions state.

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
against closed forms, paper values, special cases and brute force, EXCEPT the
GQA aggregation rule (reading Q10), which the paper does not define: it is
pinned only by its own definition plus brute force ("parity unpinned" by the
paper).
"""
from __future__ import annotations

import numpy as np

F64 = np.float64

GROUP_MAX = 0
GROUP_SUM = 1


# --------------------------------------------------------------------------
# 1. RoPE (Eq. 1; Eq. 3)
# --------------------------------------------------------------------------
def inv_freq(d: int, theta: float = 1e4) -> np.ndarray:
    """theta^(-2m/d) for m < d/2 (Eq. 1 rotation frequencies; reading Q1)."""
    if d % 2:
        raise ValueError("odd head dimension")
    m = np.arange(d // 2, dtype=F64)
    return np.power(F64(theta), -2.0 * m / d)


def rope_rotate(x, pos, freqs) -> np.ndarray:
    """x R_pos (Eq. 1): rotate each pair (x_m, x_{m+d/2}) by angle pos*freqs[m].

    Half-split pairing (reading Q2) and y1 = x1 cos - x2 sin,
    y2 = x2 cos + x1 sin (reading Q3).  ``pos`` may be an array that
    broadcasts against x[..., 0].
    """
    x = np.asarray(x, dtype=F64)
    h = x.shape[-1] // 2
    a = np.asarray(pos, dtype=F64)[..., None] * np.asarray(freqs, dtype=F64)
    c, s = np.cos(a), np.sin(a)
    x1, x2 = x[..., :h], x[..., h:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


# --------------------------------------------------------------------------
# 2. Windowed RoPE (Eq. 11; Eq. 12)
# --------------------------------------------------------------------------
def wrope_query(q, bridge: int, freqs) -> np.ndarray:
    """Post-PE query under WRoPE: q~ = q R_b (Eq. 12)."""
    return rope_rotate(q, bridge, freqs)


def wrope_key(k) -> np.ndarray:
    """Post-PE key under WRoPE: k~ = k, bitwise (Eq. 12; reading Q13)."""
    return np.asarray(k)


def wrope_score(q_i, k_j, i: int, j: int, window: int, bridge: int, freqs) -> float:
    """u_{i,j} of Eq. 11: q_i R_{i-j} k_j^T if i-j < w else q_i R_b k_j^T."""
    rel = (i - j) if (i - j) < window else bridge
    return float(np.dot(rope_rotate(q_i, rel, freqs), np.asarray(k_j, dtype=F64)))


def token_sets(n_ctx: int, window: int, n_sink: int):
    """Sinks S, window W and candidates Cand for the current token i = N-1.

    W = {j : i - j < w} = {j >= N - w} (Eq. 11 locality, reading Q5/Q7);
    S = first n_sink tokens not in W; Cand = [0, N) minus (S u W)
    (reading Q8: disjoint budget).
    """
    if n_ctx <= 0:
        raise ValueError("empty context")
    w0 = max(0, n_ctx - window)
    W = np.arange(w0, n_ctx)
    S = np.arange(0, min(n_sink, w0))
    Cand = np.arange(min(n_sink, w0), w0)
    return S, Cand, W


# --------------------------------------------------------------------------
# 3. Query-aware VQ encoding (Eq. 14; Eqs. 15-18)
# --------------------------------------------------------------------------
def qavq_encode(keys, C, H=None) -> np.ndarray:
    """s_t = argmin_j (k_t - c_j) H (k_t - c_j)^T by brute-force quadratic form.

    Eq. 14 / Eq. 20.  H = None means H = I, i.e. the
    conventional quantizer f of Eq. 5.  np.argmin returns the
    first minimum: lowest codeword index on ties (reading Q12).
    """
    keys = np.asarray(keys, dtype=F64)
    C = np.asarray(C, dtype=F64)
    Hm = np.eye(C.shape[1]) if H is None else np.asarray(H, dtype=F64)
    out = np.empty(keys.shape[0], dtype=np.int64)
    for t in range(keys.shape[0]):
        diff = keys[t][None, :] - C                       # [L, d]
        dist = np.einsum("ld,de,le->l", diff, Hm, diff)   # (k-c_j) H (k-c_j)^T
        out[t] = int(np.argmin(dist))
    return out


def qavq_encode_zspace(keys, C, H) -> np.ndarray:
    """Same code via the Cholesky reformulation (Eqs. 15-18):
    H = L L^T, z = k L, C^z = C L, f'(k; C) = f(z; C^z) = argmin ||z - c^z_j||^2."""
    keys = np.asarray(keys, dtype=F64)
    C = np.asarray(C, dtype=F64)
    Lc = np.linalg.cholesky(np.asarray(H, dtype=F64))   # lower, H = Lc Lc^T
    z = keys @ Lc
    Cz = C @ Lc
    out = np.empty(keys.shape[0], dtype=np.int64)
    for t in range(keys.shape[0]):
        diff = z[t][None, :] - Cz
        out[t] = int(np.argmin(np.sum(diff * diff, axis=1)))
    return out


def qavq_expanded_terms(C, H=None):
    """D = C H and n_j = c_j H c_j^T: (k-c_j)H(k-c_j)^T = kHk^T - 2 k.D_j + n_j
    (H symmetric).  The plain definitions of the two codebook-side terms."""
    C = np.asarray(C, dtype=F64)
    Hm = np.eye(C.shape[1]) if H is None else np.asarray(H, dtype=F64)
    D = C @ Hm
    n = np.einsum("ld,ld->l", D, C)
    return D, n


def qavq_encode_chform(keys, C, H=None) -> np.ndarray:
    """Same code via the expanded form argmin_j (n_j - 2 k.D_j)."""
    keys = np.asarray(keys, dtype=F64)
    D, n = qavq_expanded_terms(C, H)
    dist = n[None, :] - 2.0 * (keys @ D.T)
    return np.argmin(dist, axis=1).astype(np.int64)


# --------------------------------------------------------------------------
# 4. Approximate scores (Eq. 21; Eq. 6)
# --------------------------------------------------------------------------
def lut(q_rot, C) -> np.ndarray:
    """LUT[l] = q~ c_l^T for every codeword (the score table of Eq. 21)."""
    return np.asarray(q_rot, dtype=F64) @ np.asarray(C, dtype=F64).T


def approx_scores(q_rot, codes, C) -> np.ndarray:
    """u^_t = q~ c_{s_t}^T (Eq. 21), via the table then a gather by code."""
    return lut(q_rot, C)[..., np.asarray(codes, dtype=np.int64)]


def group_aggregate(scores_g, mode: int = GROUP_MAX) -> np.ndarray:
    """One ranking score per KV head from its G query heads' u^ (reading Q10)."""
    scores_g = np.asarray(scores_g, dtype=F64)
    if mode == GROUP_MAX:
        return scores_g.max(axis=0)
    if mode == GROUP_SUM:
        return scores_g.sum(axis=0)
    raise ValueError("unknown group_reduce")


# --------------------------------------------------------------------------
# 5. Top-K retrieval (readings Q8, Q11, Q12)
# --------------------------------------------------------------------------
def select_topk(agg, cand, k: int) -> np.ndarray:
    """First min(k, |Cand|) candidates by (agg desc, t asc), returned ascending."""
    cand = np.asarray(cand, dtype=np.int64)
    if k <= 0 or cand.size == 0:
        return np.zeros(0, dtype=np.int64)
    order = np.lexsort((cand, -np.asarray(agg, dtype=F64)[cand]))  # primary: -agg
    return np.sort(cand[order[: min(k, cand.size)]])


def select_topk_threshold(agg, cand, k: int) -> np.ndarray:
    """Independent second implementation: count-weighted level threshold.

    Levels v (distinct agg values over Cand) in descending order with counts
    n_v; v* = first level where the cumulative count reaches K; take every
    candidate with agg > v* plus the first m = K - #{agg > v*} (by index) with
    agg == v*.
    """
    cand = np.asarray(cand, dtype=np.int64)
    kk = min(k, cand.size)
    if kk <= 0:
        return np.zeros(0, dtype=np.int64)
    a = np.asarray(agg, dtype=F64)[cand]
    levels, counts = np.unique(a, return_counts=True)     # ascending
    levels, counts = levels[::-1], counts[::-1]
    cum = np.cumsum(counts)
    lv = int(np.searchsorted(cum, kk))                     # first cum >= kk
    vstar = levels[lv]
    above = cand[a > vstar]
    m = kk - above.size
    ties = cand[a == vstar][:m]                            # cand is ascending
    return np.sort(np.concatenate([above, ties]))


def select_topk_bruteforce(agg, cand, k: int) -> np.ndarray:
    """O(|Cand|^2) definition: t is selected iff fewer than K candidates beat
    it, where u beats t iff agg[u] > agg[t] or (agg[u] == agg[t] and u < t)."""
    cand = np.asarray(cand, dtype=np.int64)
    a = np.asarray(agg, dtype=F64)
    sel = []
    for t in cand:
        beat = 0
        for u in cand:
            if a[u] > a[t] or (a[u] == a[t] and u < t):
                beat += 1
        if beat < k:
            sel.append(int(t))
    return np.asarray(sel, dtype=np.int64)


# --------------------------------------------------------------------------
# 6. Attention over the selected rows (Eq. 2; Eq. 11)
# --------------------------------------------------------------------------
def wrope_logits(q, q_rot, keys, rows, n_ctx: int, window: int, freqs) -> np.ndarray:
    """u_j for j in rows with i = N-1: exact relative rotation q R_{i-j} k_j^T
    inside the window (i-j < w), bridge q~ k_j^T = q R_b k_j^T outside."""
    i = n_ctx - 1
    keys = np.asarray(keys, dtype=F64)
    u = np.empty(len(rows), dtype=F64)
    for n, j in enumerate(rows):
        if i - j < window:
            u[n] = np.dot(rope_rotate(q, i - j, freqs), keys[j])
        else:
            u[n] = np.dot(q_rot, keys[j])
    return u


def softmax_attention(u, V) -> np.ndarray:
    """o = Softmax(u / sqrt(d)) V (Eq. 2), with max subtraction."""
    u = np.asarray(u, dtype=F64)
    V = np.asarray(V, dtype=F64)
    x = u / np.sqrt(F64(V.shape[1]))
    p = np.exp(x - x.max())
    return (p / p.sum()) @ V


# --------------------------------------------------------------------------
# The whole decode step (P:384-397 stages (2)+(3), as SURVEY.md §8c 1-9)
# --------------------------------------------------------------------------
def decode_step_pair(q_g, keys, values, codes, C, n_ctx: int, *, window: int = 64,
                     bridge: int = 2048, n_sink: int = 4, topk: int = 0, freqs=None,
                     group_reduce: int = GROUP_MAX):
    """One (batch, KV-head) pair.

    q_g    [G, d]  pre-PE queries of the G query heads sharing this KV head
    keys   [>=N, d] pre-PE keys (= post-PE under WRoPE), values [>=N, d]
    codes  [>=N]   codeword indices s_t, C [L, d] the shared codebook
    Returns dict(out [G, d], sel [K_eff] ascending, agg [N], scores [G, N],
                 q_rot [G, d], sel_rows [|Sel|]).
    """
    q_g = np.asarray(q_g, dtype=F64)
    d = q_g.shape[1]
    if freqs is None:
        freqs = inv_freq(d)
    q_rot = wrope_query(q_g, bridge, freqs)                          # a1
    codes_n = np.asarray(codes, dtype=np.int64)[:n_ctx]
    scores = approx_scores(q_rot, codes_n, C)                        # a2+a3 [G, N]
    agg = group_aggregate(scores, group_reduce)                      # Q10
    S, Cand, W = token_sets(n_ctx, window, n_sink)
    sel = select_topk(agg, Cand, topk)                               # a4
    rows = np.concatenate([S, sel, W]).astype(np.int64)              # ascending
    out = np.empty_like(q_g)
    for g in range(q_g.shape[0]):                                    # a5+a6
        u = wrope_logits(q_g[g], q_rot[g], keys, rows, n_ctx, window, freqs)
        out[g] = softmax_attention(u, np.asarray(values, dtype=F64)[rows])
    return dict(out=out, sel=sel, agg=agg, scores=scores, q_rot=q_rot, sel_rows=rows)


def decode_step_pair_standard(q_g, keys_post, values, codes, C, n_ctx: int, *, window: int = 64,
                              n_sink: int = 4, topk: int = 0, freqs=None, group_reduce: int = GROUP_MAX):
    """One pair of the ablation configurations with standard RoPE ("Baseline" / "QAVQ"):
    the cache holds POST-PE keys k~_j = k_j R_j (RoPE, Eq. 1) and the codes quantize them;
    the query is rotated to the current position i = N-1, q~ = q R_i; approximate scores
    u^_j = q~ . c_{s_j} (Eq. 21 with the standard query), the same candidate sets and top-K rule as
    decode_step_pair (readings Q8, Q12), and every selected row -- sinks, top-K, window -- gets the
    standard logit u_j = q~ . k~_j (Eq. 2 with RoPE: no window rotation)."""
    q_g = np.asarray(q_g, dtype=F64)
    d = q_g.shape[1]
    if freqs is None:
        freqs = inv_freq(d)
    q_rot = rope_rotate(q_g, n_ctx - 1, freqs)                       # q R_i
    codes_n = np.asarray(codes, dtype=np.int64)[:n_ctx]
    scores = approx_scores(q_rot, codes_n, C)
    agg = group_aggregate(scores, group_reduce)
    S, Cand, W = token_sets(n_ctx, window, n_sink)
    sel = select_topk(agg, Cand, topk)
    rows = np.concatenate([S, sel, W]).astype(np.int64)
    kp = np.asarray(keys_post, dtype=F64)[rows]
    vr = np.asarray(values, dtype=F64)[rows]
    out = np.stack([softmax_attention(kp @ q_rot[g], vr) for g in range(q_g.shape[0])])
    return dict(out=out, sel=sel, agg=agg, scores=scores, q_rot=q_rot, sel_rows=rows)


def decode_step(q, k_cache, v_cache, codes, codebook, n_ctx: int, *, window=64, bridge=2048,
                n_sink=4, topk=0, freqs=None, group_reduce=GROUP_MAX, pairs=None):
    """Batched decode step.  q [B, Hq, d]; caches [B, Hkv, >=N, d]; codes
    [B, Hkv, >=N]; codebook [Hkv, L, d].  ``pairs`` restricts to a list of
    (b, h) pairs (sampled parity at full size); outputs for other pairs are
    left as NaN / -1."""
    q = np.asarray(q)
    B, Hq, d = q.shape
    Hkv = codebook.shape[0]
    G = Hq // Hkv
    S, Cand, W = token_sets(n_ctx, window, n_sink)
    keff = min(topk, Cand.size) if topk > 0 else 0
    out = np.full((B, Hq, d), np.nan)
    sel = np.full((B, Hkv, keff), -1, dtype=np.int64)
    if pairs is None:
        pairs = [(b, h) for b in range(B) for h in range(Hkv)]
    for b, h in pairs:
        r = decode_step_pair(q[b, h * G:(h + 1) * G], k_cache[b, h], v_cache[b, h], codes[b, h],
                             codebook[h], n_ctx, window=window, bridge=bridge, n_sink=n_sink,
                             topk=topk, freqs=freqs, group_reduce=group_reduce)
        out[b, h * G:(h + 1) * G] = r["out"]
        sel[b, h] = r["sel"]
    return out, sel


# --------------------------------------------------------------------------
# Accounting (Table 1 "Aux Mem"; sparsity P:756-759)
# --------------------------------------------------------------------------
def aux_mem_ratio(d: int, elem_bytes: int = 2, index_bytes: int = 2) -> float:
    """Index bytes per token per head / key bytes per token per head."""
    return index_bytes / (d * elem_bytes)


def sparsity_ratio(n_selected: int, n_ctx: int) -> float:
    """K/V bytes read / full-attention K/V bytes = |Sel| / N."""
    return n_selected / n_ctx
