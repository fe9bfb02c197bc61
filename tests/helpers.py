"""Shared test plumbing: run the oracle on boundary inputs, the distinct-level
gap rule of reading Q20, and the comparison metrics of readings Q18/Q19."""
from __future__ import annotations

import numpy as np
import torch

from oracle import a2ats_oracle as O

GAP = 1e-3           # BJ: K-th vs (K+1)-th score gap, read between distinct levels (Q20)
SCORE_RTOL = 1e-4    # BJ: approximate scores, row-relative (Q18)
OUT_RTOL = 2e-3      # BJ: attention output, relative L2 per (b, hq) row (Q19)


def f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").double().numpy()


def codes_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").to(torch.int64).numpy()


def cut_gap(agg: np.ndarray, cand: np.ndarray, k: int) -> float:
    """Distance from the K-th level v* to the nearest OTHER distinct level among
    the candidates (inf when K selects nothing or everything)."""
    kk = min(k, cand.size)
    if kk <= 0 or kk >= cand.size:
        return np.inf
    a = agg[cand]
    vstar = np.sort(a)[::-1][kk - 1]
    other = a[a != vstar]
    return float(np.min(np.abs(other - vstar))) if other.size else np.inf


def pair_oracle(q_g, k, v, codes, C, n_ctx, cfg, bridge=None, group_reduce=O.GROUP_MAX):
    return O.decode_step_pair(q_g, k, v, codes, C, n_ctx, window=cfg.window,
                              bridge=cfg.bridge if bridge is None else bridge, n_sink=cfg.n_sink,
                              topk=cfg.K, group_reduce=group_reduce)


def redraw_for_gap(inp: dict, cfg, n_ctx: int, seed: int, bridge=None, max_attempts: int = 40,
                   pairs=None) -> int:
    """Reading Q20 / SURVEY §8c G2: re-draw (deterministically, seed + attempt) the
    queries of every pair whose cut gap is <= GAP.  Modifies inp['q'] in place.
    Returns the number of redrawn pairs."""
    G = cfg.Hq // cfg.Hkv
    q = inp["q"]
    C = f64(inp["codebook"])
    codes = codes_np(inp["codes"])
    freqs = O.inv_freq(cfg.d)
    b_ = cfg.bridge if bridge is None else bridge
    S, cand, W = O.token_sets(n_ctx, cfg.window, cfg.n_sink)
    redrawn = 0
    pairs = pairs or [(b, h) for b in range(cfg.B) for h in range(cfg.Hkv)]
    for b, h in pairs:
        for attempt in range(max_attempts):
            qg = f64(q[b, h * G:(h + 1) * G])
            qrot = O.wrope_query(qg, b_, freqs)
            agg = O.group_aggregate(O.approx_scores(qrot, codes[b, h, :n_ctx], C[h]))
            if cut_gap(agg, cand, cfg.K) > GAP:
                break
            g = torch.Generator(device="cpu").manual_seed(seed * 1000003 + (b * 131 + h) * 977 + attempt + 1)
            new = torch.randn((G, cfg.d), generator=g).to(torch.bfloat16)
            q[b, h * G:(h + 1) * G] = new.to(q.device)
            redrawn += 1
        else:
            raise RuntimeError("could not draw a query with a clean cut")
    return redrawn


def rel_l2(x: np.ndarray, y: np.ndarray) -> float:
    return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))


def row_rel_max(x: np.ndarray, y: np.ndarray) -> float:
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))
