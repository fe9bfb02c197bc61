"""Sequence-sharded decode step across ranks (the paper
itself is single-GPU).

Rank r holds, for every (b, KV head), the global tokens [bounds[r], bounds[r+1])
in its own K/V/code arrays (local index = global index - bounds[r]); q, the
codebook and the shard STATE are replicated.  The state -- the global code
histogram, every rank's code histogram, the codes of the sinks and of the
latest tokens -- lets every rank derive the exact global top-K threshold and its
own share of the ties with no exchange (collective-free exact top-K, §8f.1).
Each decode step is ONE call into liba2ats.so (a2ats_decode_step_sharded): a0 on
the new token's owner, the LUT, the local selection and attention, one NCCL
all-gather of the partials (m, l, o) and the new token's code, the log-sum-exp
combine and the state update, all on the caller's stream (graph-capturable).
This module holds no collectives: only the communicator bootstrap (the NCCL
unique id travels through torch.distributed) and buffer ownership.
"""
from __future__ import annotations

from . import binding as _b


def shard_ranges(n_tokens: int, world: int):
    """Contiguous, balanced token shards [begin, end) for ranks 0..world-1."""
    base, rem = divmod(n_tokens, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < rem else 0)
        out.append((b, e))
        b = e
    return out


def step_bounds(ranges, n_ctx: int):
    """Bounds [R+1] of a step: the prefill shards, new tokens appended to the last rank."""
    bounds = [b for b, _ in ranges] + [max(ranges[-1][1], n_ctx)]
    return bounds


def comm_from_torch(world: int, rank: int, group=None):
    """NCCL communicator of liba2ats.so; the 128-byte unique id is broadcast from rank 0
    through torch.distributed (plumbing only)."""
    import torch.distributed as dist
    obj = [_b.a2ats_comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    return _b.a2ats_comm_init(obj[0], world, rank)


class ShardedDecoder:
    """One rank's buffers for the sharded step: prepared codebook terms, local codes, the
    replicated shard state, the workspace and (world > 1) the communicator."""

    def __init__(self, B, Hq, Hkv, L, n_max_local, codebook, H, params: _b.Params, world: int, rank: int,
                 comm=None, device="cuda", stream=None):
        import torch
        self.world, self.rank, self.comm, self.stream = world, rank, comm, stream
        self.device = torch.device(device)
        self.shape = _b.make_shape(B, Hq, Hkv, 128, L, n_max_local)
        self.params = params
        self.codebook = codebook.contiguous()
        self.nrm = torch.empty((Hkv, L), dtype=torch.float32, device=self.device)
        self.chat = torch.empty((Hkv, L, 256), dtype=torch.bfloat16, device=self.device)
        _b.a2ats_qavq_prepare(self.shape, self.codebook, None if H is None else H.contiguous().float(), self.nrm,
                              self.chat, stream)
        self.codes = torch.zeros((B, Hkv, n_max_local), dtype=torch.uint16, device=self.device)
        self.state = torch.zeros(_b.a2ats_shard_state_bytes(self.shape, params, world), dtype=torch.uint8,
                                 device=self.device)
        self.ws = torch.zeros(_b.a2ats_shard_workspace_bytes(self.shape, params, world), dtype=torch.uint8,
                              device=self.device)
        self.ws_enc = torch.zeros(_b.a2ats_build_codes_workspace_bytes(self.shape), dtype=torch.uint8,
                                  device=self.device)

    def encode(self, k_local, t_begin: int, t_end: int):
        """a0 for local tokens [t_begin, t_end) (prefill of this rank's shard)."""
        _b.a2ats_build_codes(self.shape, k_local, t_begin, t_end, self.chat, self.nrm, self.codes, None, self.ws_enc,
                             self.stream)

    def build_state(self, bounds, n_tokens: int):
        """Replicated state of tokens [0, n_tokens) (NCCL all-reduces inside the library)."""
        _b.a2ats_shard_state_build(self.shape, self.params, self.world, self.rank, bounds, n_tokens, self.codes,
                                   self.state, self.ws, self.comm, self.stream)

    def step(self, n_ctx: int, bounds, q, k_local, v_local, out, sel_out=None):
        """One decode step (token n_ctx - 1 already in its owner's K/V cache)."""
        _b.a2ats_decode_step_sharded(self.shape, self.params, n_ctx, self.world, self.rank, bounds, q, k_local,
                                     v_local, self.codes, self.codebook, self.chat, self.nrm, self.state, out,
                                     sel_out, self.ws, self.comm, self.stream)
        return out

    # the two halves around the all-gather (single-process rank simulation in tests)
    def partial(self, n_ctx: int, bounds, q, k_local, v_local, msg, sel_out=None):
        _b.a2ats_shard_step_partial(self.shape, self.params, n_ctx, self.world, self.rank, bounds, q, k_local,
                                    v_local, self.codes, self.codebook, self.chat, self.nrm, self.state, msg, sel_out,
                                    self.ws, self.stream)

    def finish(self, n_ctx: int, bounds, msgs, out):
        _b.a2ats_shard_step_finish(self.shape, self.params, n_ctx, self.world, bounds, msgs, self.state, out,
                                   self.stream)
        return out

    def close(self):
        if self.comm is not None:
            _b.a2ats_comm_destroy(self.comm)
            self.comm = None
