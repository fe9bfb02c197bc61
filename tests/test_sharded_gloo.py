"""world_size-2 gloo test of the sequence-sharded protocol on CPU.

The protocol a2ats_decode_step_sharded implements on GPUs, with its collectives run for
real over torch.distributed/gloo in two processes and the per-rank arithmetic replaced by
a numpy model built on the fp64 oracle's primitives:
  prefill   replicated state = all-reduce(SUM) of the ranks' contributions (global and
            per-rank code histograms of tokens [0, n), codes of the sinks and latest tokens);
  each step (new token n-1 on the last rank): the global K-th level v* and tie quota m
            and this rank's tie share from the state alone (no exchange); local selection
            and attention partial (m, l, o); ONE all-gather of (partial, new code); LSE
            combine in rank order; the new code joins the state on every rank.
Three steps run; the combined output and the union of the ranks' selections must equal the
unsharded oracle decode step at every context length, including cross-rank integer ties."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import a2ats_oracle as O
from paper_2502_12665_b200.sharded import shard_ranges, step_bounds

D, G, N, L, K, W, NS, STEPS = 16, 2, 300, 12, 40, 16, 4, 3


def make_problem(seed=0):
    rng = np.random.default_rng(seed)
    C = rng.integers(-3, 4, (L, D)).astype(np.float64)       # integer codebook: exact cross-code ties
    codes = rng.integers(0, L, N)
    K_ = C[codes] + 0.05 * rng.standard_normal((N, D))
    V = rng.standard_normal((N, D))
    q = rng.integers(-3, 4, (G, D)).astype(np.float64)
    return q, K_, V, codes, C


class RankModel:
    """Per-rank numpy model of the library's sharded step (B = Hkv = 1)."""

    def __init__(self, rank, world, C, codes_local, lo, bridge=0):
        self.rank, self.world, self.C, self.bridge = rank, world, C, bridge
        self.codes, self.lo = codes_local, lo                 # local codes (index = global - lo)
        self.freqs = O.inv_freq(D)

    def contribution(self, bounds, n):
        hg = np.zeros(L, np.int64)
        hr = np.zeros((self.world, L), np.int64)
        codes_g = np.full(n, -1, np.int64)                    # codes of the tokens this rank holds
        for t in range(bounds[self.rank], min(bounds[self.rank + 1], n)):
            c = self.codes[t - self.lo]
            hg[c] += 1
            hr[self.rank, c] += 1
            codes_g[t] = c
        return hg, hr, codes_g

    def partial(self, n, bounds, state, q, k_local, v_local, new_code):
        hg, hr, codes_g = state                               # replicated: tokens [0, n-1)
        owner = lambda t: int(np.searchsorted(bounds, t, side="right")) - 1
        S, cand, Wn = O.token_sets(n, W, NS)
        stat = [t for t in np.concatenate([S, Wn]) if t != n - 1]
        cnt = hg.copy()
        cnt_r = hr.copy()
        for t in stat:
            cnt[codes_g[t]] -= 1
            cnt_r[owner(t), codes_g[t]] -= 1
        qrot = O.wrope_query(q, self.bridge, self.freqs)
        agg = O.group_aggregate(O.lut(qrot, self.C))
        keff = min(K, int(cnt.sum()))
        levels = np.unique(agg[cnt > 0])[::-1]
        cum = np.cumsum([cnt[agg == v].sum() for v in levels])
        vstar = levels[int(np.searchsorted(cum, keff))]
        m = keff - int(cnt[agg > vstar].sum())
        before = int(sum(cnt_r[r][agg == vstar].sum() for r in range(self.rank)))
        e_loc = int(cnt_r[self.rank][agg == vstar].sum())
        m_loc = min(max(m - before, 0), e_loc)
        lo, hi = bounds[self.rank], bounds[self.rank + 1]
        mine = cand[(cand >= lo) & (cand < hi)]
        a = agg[self.codes[mine - self.lo]]
        self.sel = np.sort(np.concatenate([mine[a > vstar], mine[a == vstar][:m_loc]]))
        rows = np.concatenate([S, self.sel, Wn])
        rows = rows[(rows >= lo) & (rows < hi)]
        part = np.zeros((G, 130))
        for g in range(G):
            if len(rows) == 0:
                part[g, 0] = -np.inf
                continue
            u = np.array([np.dot(O.rope_rotate(q[g], n - 1 - j, self.freqs), k_local[j - self.lo]) if n - 1 - j < W
                          else np.dot(qrot[g], k_local[j - self.lo]) for j in rows]) / np.sqrt(D)
            mx = u.max()
            p = np.exp(u - mx)
            part[g, 0], part[g, 1] = mx, p.sum()
            part[g, 2:2 + D] = p @ v_local[rows - self.lo]
        msg = np.zeros(G * 130 + 1)
        msg[:G * 130] = part.ravel()
        msg[-1] = new_code if self.rank == owner(n - 1) else -1
        return msg


def combine(msgs):
    P = msgs[:, :G * 130].reshape(-1, G, 130)                # [R, G, 130]
    M = P[:, :, 0].max(axis=0)
    w = np.where(np.isneginf(P[:, :, 0]), 0.0, np.exp(P[:, :, 0] - M))
    num = (w[..., None] * P[:, :, 2:2 + D]).sum(axis=0)
    den = (w * P[:, :, 1]).sum(axis=0)
    return num / den[..., None]


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, Kc, Vc, codes, C = make_problem()
    n_pre = N - STEPS
    ranges = shard_ranges(n_pre, world)
    lo = ranges[rank][0]
    hi_all = N if rank == world - 1 else ranges[rank][1]     # new tokens join the last rank
    model = RankModel(rank, world, C, codes[lo:hi_all], lo)
    # prefill state: all-reduce of the ranks' contributions
    hg, hr, cg = model.contribution(step_bounds(ranges, n_pre), n_pre)
    t = [torch.from_numpy(hg), torch.from_numpy(hr), torch.from_numpy(cg + 1)]
    for x in t:
        dist.all_reduce(x)
    state = (t[0].numpy(), t[1].numpy(), t[2].numpy() - 1)
    results = []
    for s in range(STEPS):
        n = n_pre + s + 1
        bounds = step_bounds(ranges, n)
        new_code = codes[n - 1]                               # a0 on the owner (the oracle encodes the same key)
        msg = torch.from_numpy(model.partial(n, bounds, state, q, Kc[lo:hi_all], Vc[lo:hi_all], new_code))
        gathered = [torch.empty_like(msg) for _ in range(world)]
        dist.all_gather(gathered, msg)                        # the step's only collective
        msgs = torch.stack(gathered).numpy()
        out = combine(msgs)
        code = int(msgs[world - 1, -1])                       # state update from the owner's message
        hg, hr, cg = state
        hg, hr = hg.copy(), hr.copy()
        hg[code] += 1
        hr[world - 1, code] += 1
        cg = np.concatenate([cg, [code]])
        state = (hg, hr, cg)
        sels = [None] * world
        dist.all_gather_object(sels, model.sel.tolist())
        results.append((out, np.array(sorted(sum(sels, [])))))
    if rank == 0:
        np.savez(result_path, **{f"out{i}": r[0] for i, r in enumerate(results)},
                 **{f"sel{i}": r[1] for i, r in enumerate(results)}, hg=state[0])
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_protocol_equals_unsharded_oracle(world, tmp_path):
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    res = np.load(path)
    q, Kc, Vc, codes, C = make_problem()
    for s in range(STEPS):
        n = N - STEPS + s + 1
        ref = O.decode_step_pair(q, Kc, Vc, codes, C, n, window=W, bridge=0, n_sink=NS, topk=K)
        np.testing.assert_array_equal(res[f"sel{s}"], ref["sel"])   # exact global top-K incl. cross-rank ties
        np.testing.assert_allclose(res[f"out{s}"], ref["out"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(res["hg"], np.bincount(codes[:N], minlength=L))


def test_shard_helpers():
    assert shard_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert shard_ranges(131072, 8)[7] == (114688, 131072)
    assert step_bounds([(0, 4), (4, 7), (7, 10)], 12) == [0, 4, 7, 12]
