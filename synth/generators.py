"""Seeded input generators.

Families (SURVEY.md §8c "Input families"):
  g1  integer-exact: q and codebook entries are integers in [-8, 8]; keys are
      exactly their codewords.  With bridge b = 0 every LUT value is an integer
      representable in fp32, so cross-code score ties are exact on both sides.
  g2  realistic: q, C ~ N(0, 1) in bf16; keys = c_{z_t} + 0.1 eps (VQ
      structure of P:107-135: keys cluster around codewords); V ~ N(0, 1).
  needle: g2 plus, per (b, h), a few planted tokens whose keys are a large
      multiple of the query direction, so attention mass concentrates in the
      retrieved set (mirrors RULER retrieval).
Code usage z_t: "uniform" or "zipf" (p_l ~ (l+1)^-1.1, randomly permuted per
head).  H (query second moment, Fig. 2 / P:248-252): A A^T / d + 0.01 I.

Everything is drawn from a torch.Generator on the requested device; the same
tensors are then handed to both the oracle and the CUDA path.
"""
from __future__ import annotations

import torch

BF16 = torch.bfloat16


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


def make_codebook(Hkv: int, L: int, d: int, family: str, g: torch.Generator, device) -> torch.Tensor:
    if family == "g1":
        return torch.randint(-8, 9, (Hkv, L, d), generator=g, device=device).to(BF16)
    return torch.randn((Hkv, L, d), generator=g, device=device).to(BF16)


def make_query(B: int, Hq: int, d: int, family: str, g: torch.Generator, device) -> torch.Tensor:
    if family == "g1":
        return torch.randint(-8, 9, (B, Hq, d), generator=g, device=device).to(BF16)
    return torch.randn((B, Hq, d), generator=g, device=device).to(BF16)


def make_h(Hkv: int, d: int, g: torch.Generator, device) -> torch.Tensor:
    A = torch.randn((Hkv, d, d), generator=g, device=device, dtype=torch.float32)
    H = A @ A.transpose(1, 2) / d + 0.01 * torch.eye(d, device=device)
    return 0.5 * (H + H.transpose(1, 2))


def make_codes(B: int, Hkv: int, n: int, L: int, dist: str, g: torch.Generator, device) -> torch.Tensor:
    """z [B, Hkv, n] int32: the codeword each synthetic key is drawn around."""
    if dist == "uniform":
        return torch.randint(0, L, (B, Hkv, n), generator=g, device=device, dtype=torch.int32)
    if dist == "zipf":
        p = torch.arange(1, L + 1, device=device, dtype=torch.float64).pow(-1.1)
        out = torch.empty((B, Hkv, n), dtype=torch.int32, device=device)
        for h in range(Hkv):
            perm = torch.randperm(L, generator=g, device=device)
            idx = torch.multinomial(p, B * n, replacement=True, generator=g)
            out[:, h] = perm[idx].view(B, n).to(torch.int32)
        return out
    raise ValueError(dist)


def make_inputs(cfg, seed: int, device="cpu", family: str = "g2", code_dist: str = "uniform",
                n_max: int | None = None, with_h: bool = True, n_needles: int = 4, codebook=None) -> dict:
    """All boundary inputs for one config.  Keys/values are drawn for n_max
    tokens (>= cfg.N) so appended decode steps have rows to read.  codebook: a given
    (replicated) codebook the keys cluster around instead of a fresh draw (sharded runs)."""
    device = torch.device(device)
    g = _gen(seed, device)
    n_max = cfg.n_max() if n_max is None else n_max
    C = make_codebook(cfg.Hkv, cfg.L, cfg.d, family, g, device)
    if codebook is not None:
        C = codebook.to(device)
    q = make_query(cfg.B, cfg.Hq, cfg.d, family, g, device)
    z = make_codes(cfg.B, cfg.Hkv, n_max, cfg.L, code_dist, g, device)
    k = torch.empty((cfg.B, cfg.Hkv, n_max, cfg.d), dtype=BF16, device=device)
    v = torch.empty_like(k)
    for h in range(cfg.Hkv):              # per head keeps the peak temporary small
        zh = z[:, h].reshape(-1).long()
        base = C[h].index_select(0, zh).view(cfg.B, n_max, cfg.d)
        if family == "g1":
            k[:, h] = base
        else:
            noise = torch.randn((cfg.B, n_max, cfg.d), generator=g, device=device, dtype=torch.float32)
            k[:, h] = (base.float() + 0.1 * noise).to(BF16)
        v[:, h] = torch.randn((cfg.B, n_max, cfg.d), generator=g, device=device,
                              dtype=torch.float32).to(BF16)
    if family == "needle":
        # plant n_needles tokens per pair at random candidate positions whose key
        # is 4x the first query head of the group (not a codeword: its code is z).
        G = cfg.Hq // cfg.Hkv
        lo, hi = cfg.n_sink, max(cfg.n_sink + 1, cfg.N - cfg.window)
        pos = torch.randint(lo, hi, (cfg.B, cfg.Hkv, n_needles), generator=g, device=device)
        for b in range(cfg.B):
            for h in range(cfg.Hkv):
                k[b, h, pos[b, h]] = (4.0 * q[b, h * G].float()).to(BF16)
    out = dict(q=q, k_cache=k, v_cache=v, z=z, codebook=C, n_max=n_max)
    if with_h:
        out["H"] = make_h(cfg.Hkv, cfg.d, g, device)
    return out
