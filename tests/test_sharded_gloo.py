"""world_size-2 gloo test of the sequence-sharded decode orchestration
(paper_2502_12665_b200/sharded.py) on CPU.

The collective sequence (all_reduce of candidate histograms, all_gather of
per-rank tie counts, all_gather of partial (m, l, o), LSE combine in rank
order) runs for real over torch.distributed/gloo in two processes; the four
per-rank kernels are replaced by a numpy stand-in built on the fp64 oracle's
primitives.  The combined output and the union of per-rank selections must
equal the unsharded oracle decode step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import a2ats_oracle as O
from paper_2502_12665_b200.sharded import ShardStep, shard_ranges, tie_offsets

D, G, N, L, K, W, NS = 16, 2, 300, 12, 40, 16, 4


def make_problem(seed=0):
    rng = np.random.default_rng(seed)
    C = rng.integers(-3, 4, (L, D)).astype(np.float64)       # integer codebook: exact cross-code ties
    codes = rng.integers(0, L, N)
    K_ = C[codes] + 0.05 * rng.standard_normal((N, D))
    V = rng.standard_normal((N, D))
    q = rng.integers(-3, 4, (G, D)).astype(np.float64)
    return q, K_, V, codes, C


class NumpyShardKernels:
    """Per-rank stand-in for the C-ABI shard kernels (B = Hkv = 1)."""

    def __init__(self, C, bridge=0):
        self.C, self.bridge = C, bridge
        self.freqs = O.inv_freq(D)

    def hist(self, n_ctx, sb, sl, q, codes_local, hist_local):
        qg = q.numpy()
        self.qrot = O.wrope_query(qg, self.bridge, self.freqs)
        self.agg = O.group_aggregate(O.lut(self.qrot, self.C))           # [L]
        S, cand, Wn = O.token_sets(n_ctx, W, NS)
        mine = cand[(cand >= sb) & (cand < sb + sl)]
        self.local_cand = mine
        self.local_codes = codes_local.numpy()
        cnt = np.bincount(self.local_codes[mine - sb], minlength=L)
        self.cand_local = cnt
        return torch.from_numpy(cnt.astype(np.int32)).view(1, 1, L)

    def threshold(self, n_ctx, cand_global):
        cnt = cand_global.view(-1).numpy().astype(np.int64)
        total = int(cnt.sum())
        self.keff = min(K, total)
        levels = np.unique(self.agg[cnt > 0])[::-1]
        cum = np.cumsum([cnt[self.agg == v].sum() for v in levels])
        lv = int(np.searchsorted(cum, self.keff))
        self.vstar = levels[lv]
        self.m = self.keff - int(cnt[self.agg > self.vstar].sum())
        gt = int(self.cand_local[self.agg > self.vstar].sum())
        eq = int(self.cand_local[self.agg == self.vstar].sum())
        return torch.tensor([[[gt, eq]]], dtype=torch.int32)

    def attend(self, n_ctx, sb, sl, rank, world, counts_all, q, k_local, v_local, codes_local):
        before = int(tie_offsets(counts_all)[rank].view(-1)[0])
        eq_r = int(counts_all[rank].view(-1)[1])
        m_r = min(max(self.m - before, 0), eq_r)
        a = self.agg[self.local_codes[self.local_cand - sb]]
        above = self.local_cand[a > self.vstar]
        tied = self.local_cand[a == self.vstar][:m_r]
        self.sel = np.sort(np.concatenate([above, tied]))
        S, cand, Wn = O.token_sets(n_ctx, W, NS)
        rows = np.concatenate([S, self.sel, Wn])
        rows = rows[(rows >= sb) & (rows < sb + sl)]
        qg = q.numpy()
        kl, vl = k_local.numpy(), v_local.numpy()
        part = np.zeros((1, G, 130))
        for g in range(G):
            u = np.array([np.dot(O.rope_rotate(qg[g], n_ctx - 1 - j, self.freqs), kl[j - sb]) if n_ctx - 1 - j < W
                          else np.dot(self.qrot[g], kl[j - sb]) for j in rows]) / np.sqrt(D)
            if len(rows) == 0:
                part[0, g, 0] = -np.inf
                continue
            mx = u.max()
            p = np.exp(u - mx)
            part[0, g, 0], part[0, g, 1] = mx, p.sum()
            part[0, g, 2:2 + D] = p @ vl[rows - sb]
        return torch.from_numpy(part)

    def combine(self, parts_all, out):
        P = parts_all.numpy()                                     # [R, 1, G, 130]
        M = P[:, :, :, 0].max(axis=0)
        w = np.exp(P[:, :, :, 0] - M)
        w[np.isnan(w)] = 0.0
        num = (w[..., None] * P[:, :, :, 2:2 + D]).sum(axis=0)
        den = (w * P[:, :, :, 1]).sum(axis=0)
        out.copy_(torch.from_numpy(num / den[..., None]))
        return out


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, Kc, Vc, codes, C = make_problem()
    sb, se = shard_ranges(N, world)[rank]
    kern = NumpyShardKernels(C)
    step = ShardStep(kern, rank, world)
    out = torch.zeros((1, G, D), dtype=torch.float64)
    step(N, sb, se - sb, torch.from_numpy(q), torch.from_numpy(Kc[sb:se]), torch.from_numpy(Vc[sb:se]),
         torch.from_numpy(codes[sb:se]), None, out)
    sels = [None] * world
    dist.all_gather_object(sels, kern.sel.tolist())
    if rank == 0:
        np.savez(result_path, out=out.numpy(), sel=np.array(sorted(sum(sels, []))))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_step_equals_unsharded_oracle(world, tmp_path):
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    res = np.load(path)
    q, Kc, Vc, codes, C = make_problem()
    ref = O.decode_step_pair(q, Kc, Vc, codes, C, N, window=W, bridge=0, n_sink=NS, topk=K)
    np.testing.assert_array_equal(res["sel"], ref["sel"])      # exact global top-K incl. cross-rank ties
    np.testing.assert_allclose(res["out"][0], ref["out"], rtol=0, atol=1e-12)


def test_shard_helpers():
    assert shard_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert shard_ranges(131072, 8)[7] == (114688, 131072)
    ca = torch.tensor([[[3, 5]], [[1, 2]], [[0, 7]]])
    np.testing.assert_array_equal(tie_offsets(ca).view(-1).numpy(), [0, 5, 7])
