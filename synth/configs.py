"""Workload shapes of BASELINE.json's configs (C1-C5) -- SURVEY.md §8d.

Llama-3.1-8B and Mistral-7B attention shapes: 32 query heads, 8 KV heads,
d = 128.  WRoPE w = 64, b = 2048; 4 sinks; codebook 4096
(P:431).  Retrieval budget K = ceil(0.06 N) (reading Q9 of DESIGN.md).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace


def budget_k(n_ctx: int, frac: float = 0.06) -> int:
    """Absolute top-K for a fractional budget (reading Q9)."""
    return int(math.ceil(frac * n_ctx - 1e-9))


@dataclass(frozen=True)
class Config:
    name: str
    B: int
    Hq: int
    Hkv: int
    d: int
    N: int            # context length n_ctx (includes the current token)
    L: int            # codebook size
    K: int            # retrieved tokens (absolute)
    window: int = 64
    bridge: int = 2048
    n_sink: int = 4
    kv_host: bool = False
    note: str = ""

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv

    def n_max(self, extra: int = 0) -> int:
        n = self.N + extra
        return (n + 63) // 64 * 64   # a multiple of 64: the long-context select loads 128-B code rows by TMA

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    "C1": Config("C1", B=1, Hq=1, Hkv=1, d=128, N=4096, L=256, K=256,
                 note="1 KV head, 4K ctx, batch 1, L=256, top-K 256 + 64 window"),
    "C2": Config("C2", B=16, Hq=32, Hkv=8, d=128, N=32768, L=4096, K=budget_k(32768),
                 note="Llama-3.1-8B shapes, 32K ctx, batch 16, ~6% budget, 1xB200"),
    "C3": Config("C3", B=32, Hq=32, Hkv=8, d=128, N=65536, L=4096, K=budget_k(65536), kv_host=True,
                 note="Mistral-7B shapes, 64K ctx, batch 32, K/V in pinned host memory"),
    "C4": Config("C4", B=64, Hq=32, Hkv=8, d=128, N=131072, L=4096, K=budget_k(131072),
                 note="Llama-3.1-8B shapes, 128K ctx, batch 64 (sequence-sharded at P>1)"),
}
