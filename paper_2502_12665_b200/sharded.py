"""Sequence-sharded decode step across ranks (the paper itself is
single-GPU).

Rank r holds, for every (b, KV head), the contiguous global token range
[shard_begin, shard_begin + shard_len) of the context in its own K/V/code
arrays (local index = global index - shard_begin).  q and the codebook are
replicated.  One decode step exchanges only small, query-dependent summaries:

  1. kernels.hist       LUT (replicated, bitwise identical on every rank) and the
                        rank's candidate histogram over codewords      [B,Hkv,L] i32
  2. all_reduce(SUM)    -> global candidate histogram: every rank derives the same
                        K-th level v* and tie quota m (exact global top-K,
                        no candidate exchange)
  3. kernels.threshold  v*, m and this rank's (#above v*, #at v*)     [B,Hkv,2] i32
  4. all_gather         -> every rank knows how many tied tokens lower ranks hold
                        (ties go to the lowest global token index, reading Q12)
  5. kernels.attend     local selection + exact attention over the rank's rows of
                        Sel -> partial (m, l, o)                        [B,Hq,130] f32
  6. all_gather         -> kernels.combine: log-sum-exp combine in rank order

Collectives go through torch.distributed (NCCL on GPUs, gloo in CPU tests);
`kernels` is the C-ABI binding (or, in tests, any object with the same four
methods).  Bytes exchanged per step: 4*B*Hkv*L (allreduce) + 8*B*Hkv*R +
520*B*Hq*R, independent of the context length.
"""
from __future__ import annotations

from dataclasses import dataclass


def shard_ranges(n_tokens: int, world: int):
    """Contiguous, balanced token shards [begin, end) for ranks 0..world-1."""
    base, rem = divmod(n_tokens, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < rem else 0)
        out.append((b, e))
        b = e
    return out


def tie_offsets(counts_all):
    """counts_all[r, ..., 1] = #tied candidates on rank r; returns, per rank, the
    number of tied candidates held by lower ranks (exclusive prefix over ranks)."""
    import torch
    eq = counts_all[..., 1]
    return torch.cumsum(eq, dim=0) - eq


@dataclass
class ShardStep:
    """Collective orchestration of one sharded decode step."""
    kernels: object
    rank: int
    world: int
    group: object = None

    def __call__(self, n_ctx: int, shard_begin: int, shard_len: int, q, k_local, v_local, codes_local, hist_local,
                 out):
        import torch
        import torch.distributed as dist
        K = self.kernels
        cand = K.hist(n_ctx, shard_begin, shard_len, q, codes_local, hist_local)       # [B,Hkv,L] int32
        if self.world > 1:
            dist.all_reduce(cand, op=dist.ReduceOp.SUM, group=self.group)
        counts = K.threshold(n_ctx, cand)                                               # [B,Hkv,2] int32
        if self.world > 1:
            gathered = [torch.empty_like(counts) for _ in range(self.world)]
            dist.all_gather(gathered, counts, group=self.group)
            counts_all = torch.stack(gathered)
        else:
            counts_all = counts.unsqueeze(0)
        part = K.attend(n_ctx, shard_begin, shard_len, self.rank, self.world, counts_all, q, k_local, v_local,
                        codes_local)                                                    # [B,Hq,130] f32
        if self.world > 1:
            parts = [torch.empty_like(part) for _ in range(self.world)]
            dist.all_gather(parts, part, group=self.group)
            parts_all = torch.stack(parts)
        else:
            parts_all = part.unsqueeze(0)
        return K.combine(parts_all, out)


class GpuShardKernels:
    """The four per-rank steps of ShardStep on the C ABI (liba2ats.so)."""

    def __init__(self, B, Hq, Hkv, L, n_max_local, codebook, params, device="cuda", stream=None):
        import torch

        from . import binding as _b
        self._b = _b
        self.shape = _b.make_shape(B, Hq, Hkv, 128, L, n_max_local)
        self.params = params
        self.codebook = codebook
        self.stream = stream
        self.ws = torch.zeros(_b.a2ats_shard_workspace_bytes(self.shape, params), dtype=torch.uint8, device=device)
        self.cand = torch.empty((B, Hkv, L), dtype=torch.int32, device=device)
        self.counts = torch.empty((B, Hkv, 2), dtype=torch.int32, device=device)
        self.part = torch.empty((B, Hq, 130), dtype=torch.float32, device=device)
        self.sel_out = None

    def hist(self, n_ctx, sb, sl, q, codes_local, hist_local):
        self._b.a2ats_shard_hist(self.shape, self.params, n_ctx, sb, sl, q, codes_local, self.codebook, hist_local,
                                 self.cand, self.ws, self.stream)
        return self.cand

    def threshold(self, n_ctx, cand_global):
        self._b.a2ats_shard_threshold(self.shape, self.params, n_ctx, cand_global, self.counts, self.ws, self.stream)
        return self.counts

    def attend(self, n_ctx, sb, sl, rank, world, counts_all, q, k_local, v_local, codes_local):
        self._b.a2ats_shard_attend(self.shape, self.params, n_ctx, sb, sl, rank, world, counts_all.contiguous(), q,
                                   k_local, v_local, codes_local, self.part, self.sel_out, self.ws, self.stream)
        return self.part

    def combine(self, parts_all, out):
        self._b.a2ats_combine(self.shape, parts_all.shape[0], parts_all.contiguous(), out, self.stream)
        return out
