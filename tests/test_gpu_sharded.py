"""GPU parity of the sequence-sharded decode step on one device.

R ranks are simulated in one process through the two halves of the C entry point
a2ats_decode_step_sharded (a2ats_shard_step_partial / a2ats_shard_step_finish):
every rank has its own local K/V/code arrays, workspace and replicated state; the
step's single collective (all-gather of the messages) is replaced by its definition
(stacking), and the prefill state build's all-reduce by the sum of the ranks'
contributions.  Checked against the fp64 oracle: the union of the ranks' selections
equals the oracle's top-K exactly (ties across ranks included), every rank's output is
the same and within 2e-3 of the oracle, the new token's code (a0 on its owner) equals
the oracle's, and the state after several steps equals the state built from scratch.
"""
import numpy as np
import pytest
import torch

from helpers import OUT_RTOL, codes_np, f64, pair_oracle, redraw_for_gap, rel_l2
from oracle import a2ats_oracle as O
from synth import Config, make_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12665_b200 as A
    from paper_2502_12665_b200 import binding as Bd
    from paper_2502_12665_b200.sharded import ShardedDecoder, shard_ranges, step_bounds


def state_views(dec):
    lay = Bd.a2ats_shard_state_layout(dec.shape, dec.params, dec.world)
    P = dec.shape.B * dec.shape.Hkv
    L = dec.shape.L
    st = dec.state
    hg = st[lay["hist_g"]:lay["hist_g"] + P * L * 4].view(torch.int32)
    hr = st[lay["hist_r"]:lay["hist_r"] + dec.world * P * L * 4].view(torch.int32)
    ring = st[lay["ring"]:lay["ring"] + P * lay["WR"] * 2].view(torch.int16)
    sk = st[lay["sinkc"]:lay["sinkc"] + P * lay["n_sink_cap"] * 2].view(torch.int16)
    return [hg, hr, ring, sk]


def make_ranks(cfg, inp, ranges, n_pre, extra):
    R = len(ranges)
    n_loc = max(e - b for b, e in ranges) + extra
    n_loc = (n_loc + 63) // 64 * 64
    params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K)
    C = inp["codebook"].cuda()
    ranks = []
    for r, (b0, e0) in enumerate(ranges):
        e_all = e0 + (extra if r == R - 1 else 0)

        def local(t):
            x = torch.zeros((cfg.B, cfg.Hkv, n_loc) + tuple(t.shape[3:]), dtype=t.dtype)
            x[:, :, :e_all - b0] = t[:, :, b0:e_all]
            return x.cuda()
        dec = ShardedDecoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, n_loc, C, None, params, R, r)
        lc = local(inp["codes"])
        lc[:, :, max(0, n_pre - b0):] = 0           # tokens >= n_pre are encoded by the steps (a0)
        dec.codes.copy_(lc)
        ranks.append(dict(dec=dec, b=b0, k=local(inp["k_cache"]), v=local(inp["v_cache"])))
    # prefill state: the all-reduce of the ranks' contributions, by definition
    bounds0 = step_bounds(ranges, n_pre)
    for rk in ranks:
        rk["dec"].build_state(bounds0, n_pre)
    torch.cuda.synchronize()
    views = [state_views(rk["dec"]) for rk in ranks]
    summed = [sum(v[i].to(torch.int64) for v in views) for i in range(4)]
    for v in views:
        for i in range(4):
            v[i].copy_(summed[i].to(v[i].dtype))
    return ranks


def sharded_step(cfg, ranks, ranges, n_ctx, q):
    R = len(ranks)
    bounds = step_bounds(ranges, n_ctx)
    msg_f = Bd.a2ats_shard_msg_bytes(ranks[0]["dec"].shape) // 4
    msgs = torch.empty((R, msg_f), dtype=torch.float32, device="cuda")
    sels = []
    for r, rk in enumerate(ranks):
        sel = torch.full((cfg.B, cfg.Hkv, max(cfg.K, 1)), -1, dtype=torch.int32, device="cuda")
        rk["dec"].partial(n_ctx, bounds, q, rk["k"], rk["v"], msgs[r], sel_out=sel)
        sels.append(sel)
    outs = []
    for rk in ranks:
        out = torch.empty((cfg.B, cfg.Hq, 128), device="cuda")
        rk["dec"].finish(n_ctx, bounds, msgs, out)
        outs.append(out)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs], [s.cpu().numpy() for s in sels]


def check_step(cfg, inp, outs, sels, n_ctx, ref_codes):
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])     # every rank holds the same combined output
    G = cfg.Hq // cfg.Hkv
    C = f64(inp["codebook"])
    for b in range(cfg.B):
        for h in range(cfg.Hkv):
            r = pair_oracle(f64(inp["q"][b, h * G:(h + 1) * G]), f64(inp["k_cache"][b, h]),
                            f64(inp["v_cache"][b, h]), ref_codes[b, h], C[h], n_ctx, cfg.with_(N=n_ctx))
            got = sorted(int(x) for s in sels for x in s[b, h] if x >= 0)
            np.testing.assert_array_equal(got, r["sel"], err_msg=f"pair {(b, h)} at n = {n_ctx}")
            for g in range(G):
                e = rel_l2(outs[0][b, h * G + g], r["out"][g])
                assert e <= OUT_RTOL, (b, h, g, e)


def run_case(cfg, inp, ranges, steps=1):
    """Prefill [0, N - steps), then `steps` sharded decode steps ending at n = N."""
    N = cfg.N
    n_pre = N - steps
    ranks = make_ranks(cfg, inp, ranges, n_pre, extra=steps + 8)
    ref_codes = codes_np(inp["codes"]).copy()
    keys = f64(inp["k_cache"])
    for s in range(steps):
        n = n_pre + s + 1
        for b in range(cfg.B):                        # the oracle's code of the new token (a0, Eq. 14)
            for h in range(cfg.Hkv):
                ref_codes[b, h, n - 1] = O.qavq_encode(keys[b, h, n - 1:n], f64(inp["codebook"])[h])[0]
        outs, sels = sharded_step(cfg, ranks, ranges, n, inp["q"].cuda())
        own = ranks[-1]
        got = own["dec"].codes[:, :, n - 1 - own["b"]].cpu().to(torch.int64).numpy()
        np.testing.assert_array_equal(got, ref_codes[:, :, n - 1])   # a0 on the owner == the oracle
        check_step(cfg, inp, outs, sels, n, ref_codes)
    # the state after the steps == the state of the final codes (the ranks' codes are the oracle's)
    views = [state_views(rk["dec"]) for rk in ranks]
    for v in views[1:]:
        for i in range(4):
            assert torch.equal(v[i], views[0][i])
    P = cfg.B * cfg.Hkv
    hg = views[0][0].view(P, cfg.L).cpu().numpy()
    want = np.stack([np.bincount(ref_codes[b, h, :N], minlength=cfg.L) for b in range(cfg.B) for h in range(cfg.Hkv)])
    np.testing.assert_array_equal(hg, want)
    hr = views[0][1].view(len(ranges), P, cfg.L).cpu().numpy()
    bounds = step_bounds(ranges, N)
    for r in range(len(ranges)):
        want_r = np.stack([np.bincount(ref_codes[b, h, bounds[r]:bounds[r + 1]], minlength=cfg.L)
                           for b in range(cfg.B) for h in range(cfg.Hkv)])
        np.testing.assert_array_equal(hr[r], want_r)


SH = Config("shard", B=2, Hq=8, Hkv=2, d=128, N=40001, L=1000, K=2400)


def prepared(cfg, seed, **kw):
    inp = make_inputs(cfg, seed, device="cpu", with_h=False, **kw)
    inp["codes"] = inp["z"].to(torch.uint16)
    return inp


@pytest.mark.parametrize("R", [1, 2, 3, 4])
def test_sharded_matches_oracle(R):
    inp = prepared(SH, 201 + R)
    redraw_for_gap(inp, SH, SH.N, 201 + R)
    run_case(SH, inp, shard_ranges(SH.N - 1, R))


def test_sharded_three_steps_state_update():
    inp = prepared(SH, 231)
    for n in (SH.N - 2, SH.N - 1, SH.N):
        redraw_for_gap(inp, SH.with_(N=n), n, 231 + n)
    run_case(SH, inp, shard_ranges(SH.N - 3, 3), steps=3)


def test_sharded_integer_ties_across_ranks():
    cfg = SH.with_(L=300, K=5000, bridge=0)
    inp = prepared(cfg, 211, family="g1", code_dist="zipf")
    run_case(cfg, inp, shard_ranges(cfg.N - 1, 3))


def test_sharded_window_and_sinks_straddle_ranks():
    inp = prepared(SH, 221)
    redraw_for_gap(inp, SH, SH.N, 221)
    N = SH.N
    run_case(SH, inp, [(0, 2), (2, N - 31), (N - 31, N - 1)])


def test_sharded_rank_without_candidates():
    """A middle rank holding only a few tokens (and one holding none)."""
    inp = prepared(SH, 241)
    redraw_for_gap(inp, SH, SH.N, 241)
    N = SH.N
    run_case(SH, inp, [(0, 20000), (20000, 20000), (20000, 20010), (20010, N - 1)])


def test_full_entry_point_with_nccl_comm():
    """a2ats_comm_unique_id / a2ats_comm_init (NCCL loaded by the library) and the one-call
    a2ats_decode_step_sharded at one rank (state built by a2ats_shard_state_build with the
    communicator), two steps: selection and output equal to the oracle's; a2ats_comm_destroy."""
    from paper_2502_12665_b200.sharded import comm_from_torch
    cfg = SH.with_(N=20001, K=1200)
    inp = prepared(cfg, 251)
    for n in (cfg.N - 1, cfg.N):
        redraw_for_gap(inp, cfg.with_(N=n), n, 251 + n)
    n_pre = cfg.N - 2
    n_loc = (cfg.N + 8 + 63) // 64 * 64
    params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K)
    comm = comm_from_torch(1, 0)
    dec = ShardedDecoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, n_loc, inp["codebook"].cuda(), None, params, 1, 0, comm)
    kc = torch.zeros((cfg.B, cfg.Hkv, n_loc, 128), dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    kc[:, :, :cfg.N] = inp["k_cache"][:, :, :cfg.N]
    vc[:, :, :cfg.N] = inp["v_cache"][:, :, :cfg.N]
    kc, vc = kc.cuda(), vc.cuda()
    lc = torch.zeros((cfg.B, cfg.Hkv, n_loc), dtype=torch.uint16)
    lc[:, :, :n_pre] = inp["codes"][:, :, :n_pre]
    dec.codes.copy_(lc.cuda())
    dec.build_state([0, n_pre], n_pre)
    ref_codes = codes_np(inp["codes"]).copy()
    keys = f64(inp["k_cache"])
    for n in (cfg.N - 1, cfg.N):
        for b in range(cfg.B):
            for h in range(cfg.Hkv):
                ref_codes[b, h, n - 1] = O.qavq_encode(keys[b, h, n - 1:n], f64(inp["codebook"])[h])[0]
        out = torch.empty((cfg.B, cfg.Hq, 128), device="cuda")
        sel = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
        dec.step(n, [0, n], inp["q"].cuda(), kc, vc, out, sel_out=sel)
        torch.cuda.synchronize()
        check_step(cfg.with_(N=n), inp, [out.cpu().numpy()], [sel.cpu().numpy()], n, ref_codes)
    dec.close()
