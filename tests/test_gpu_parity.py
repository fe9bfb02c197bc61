"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle, element by
element, on the same seeded inputs (BJ tolerances: codes and top-K sets
bit-exact, scores 1e-4 row-relative, output 2e-3 relative L2)."""
import numpy as np
import pytest
import torch

from helpers import OUT_RTOL, SCORE_RTOL, codes_np, cut_gap, f64, pair_oracle, redraw_for_gap, rel_l2, row_rel_max
from oracle import a2ats_oracle as O
from synth import CONFIGS, Config, make_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12665_b200 as A


def hist_of(codes: torch.Tensor, L: int, n_ctx: int) -> torch.Tensor:
    B, Hkv, _ = codes.shape
    c = codes[:, :, :n_ctx].to(torch.int64)
    h = torch.zeros((B, Hkv, L), dtype=torch.int32, device=codes.device)
    h.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
    return h


def run_case(cfg: Config, seed: int, family="g2", code_dist="uniform", bridge=None, n_ctx=None, use_hist=True,
             scores=True, gap_redraw=True, group_reduce=O.GROUP_MAX, pairs=None, device="cuda", n_max=None,
             lut_engine=0):
    n_ctx = cfg.N if n_ctx is None else n_ctx
    bridge = cfg.bridge if bridge is None else bridge
    inp = make_inputs(cfg, seed, device="cpu", family=family, code_dist=code_dist, with_h=False, n_max=n_max)
    inp["codes"] = inp["z"].to(torch.uint16)
    if gap_redraw and family != "g1":
        redraw_for_gap(inp, cfg.with_(bridge=bridge), n_ctx, seed, pairs=pairs)
    dev = {k: (v.to(device) if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(window=cfg.window, bridge=bridge, n_sink=cfg.n_sink, topk=cfg.K, group_reduce=group_reduce,
                      lut_engine=lut_engine)
    shape = A.make_shape(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.L, inp["n_max"])
    ws = torch.zeros(A.a2ats_decode_workspace_bytes(shape, params), dtype=torch.uint8, device=device)
    out = torch.full((cfg.B, cfg.Hq, cfg.d), float("nan"), device=device)
    S, cand, W = O.token_sets(n_ctx, cfg.window, cfg.n_sink)
    keff = min(cfg.K, cand.size)
    sel = torch.full((cfg.B, cfg.Hkv, max(keff, 1)), -1, dtype=torch.int32, device=device)
    sc = torch.empty((cfg.B, cfg.Hq, n_ctx), device=device) if scores else None
    hist = hist_of(dev["codes"], cfg.L, n_ctx) if use_hist else None
    A.a2ats_decode_step(shape, params, n_ctx, dev["q"], dev["k_cache"], dev["v_cache"], dev["codes"],
                        dev["codebook"], hist, out, sel, sc, ws)
    torch.cuda.synchronize()
    return inp, dict(out=out.cpu().numpy(), sel=sel.cpu().numpy()[:, :, :keff], scores=None if sc is None else sc.cpu().numpy(),
                     ws=ws), params


def check_against_oracle(cfg, inp, gpu, n_ctx=None, bridge=None, pairs=None, exact_sets=True,
                         group_reduce=O.GROUP_MAX):
    n_ctx = cfg.N if n_ctx is None else n_ctx
    G = cfg.Hq // cfg.Hkv
    C = f64(inp["codebook"])
    codes = codes_np(inp["codes"])
    pairs = pairs or [(b, h) for b in range(cfg.B) for h in range(cfg.Hkv)]
    worst = dict(score=0.0, out=0.0)
    for b, h in pairs:
        r = pair_oracle(f64(inp["q"][b, h * G:(h + 1) * G]), f64(inp["k_cache"][b, h]), f64(inp["v_cache"][b, h]),
                        codes[b, h], C[h], n_ctx, cfg, bridge=bridge, group_reduce=group_reduce)
        if exact_sets:
            np.testing.assert_array_equal(gpu["sel"][b, h], r["sel"], err_msg=f"top-K set of pair {(b, h)}")
        if gpu["scores"] is not None:
            for g in range(G):
                e = row_rel_max(gpu["scores"][b, h * G + g], r["scores"][g])
                worst["score"] = max(worst["score"], e)
                assert e <= SCORE_RTOL, f"scores row {(b, h * G + g)} rel err {e}"
        for g in range(G):
            e = rel_l2(gpu["out"][b, h * G + g], r["out"][g])
            worst["out"] = max(worst["out"], e)
            assert e <= OUT_RTOL, f"output row {(b, h * G + g)} rel L2 {e}"
    return worst


# ------------------------------------------------------------------ C1 and small multi-tile shapes
# LUT engines (a2): AUTO (FMA for B*G <= 8, reading Q26), forced tensor cores, forced FMA
ENGINES = [0, 1, 2]


@pytest.mark.parametrize("lut_engine", ENGINES)
def test_c1_realistic(lut_engine):
    cfg = CONFIGS["C1"]
    inp, gpu, _ = run_case(cfg, seed=11, lut_engine=lut_engine)
    w = check_against_oracle(cfg, inp, gpu)
    assert w["out"] < 1e-4


@pytest.mark.parametrize("lut_engine", ENGINES)
def test_c1_integer_exact_ties(lut_engine):
    # G1 family with b = 0: LUT values exact in fp32 -> cross-code ties exact on both sides
    cfg = CONFIGS["C1"]
    inp, gpu, _ = run_case(cfg, seed=12, family="g1", bridge=0, lut_engine=lut_engine)
    check_against_oracle(cfg, inp, gpu, bridge=0)


SMALL = Config("small", B=2, Hq=8, Hkv=2, d=128, N=20001, L=1000, K=1200)


@pytest.mark.parametrize("use_hist", [True, False])
def test_multi_tile_ragged(use_hist):
    inp, gpu, _ = run_case(SMALL, seed=21, use_hist=use_hist)
    check_against_oracle(SMALL, inp, gpu)


@pytest.mark.parametrize("lut_engine", [1, 2])
def test_multi_tile_integer_ties_gqa(lut_engine):
    cfg = SMALL.with_(L=300, K=5000)
    inp, gpu, _ = run_case(cfg, seed=22, family="g1", bridge=0, code_dist="zipf", lut_engine=lut_engine)
    check_against_oracle(cfg, inp, gpu, bridge=0)


LONG = Config("long", B=2, Hq=8, Hkv=2, d=128, N=70001, L=1000, K=4200)


@pytest.mark.parametrize("use_hist", [True, False])
def test_long_context_chunked_select(use_hist):
    # 3 code chunks per pair (n_max % 16 == 8: odd rows start 16 B past a 32-B boundary):
    # streaming select with hist, threshold kernel + chunked scan with the cross-chunk
    # look-back without
    inp, gpu, _ = run_case(LONG, seed=23, use_hist=use_hist, scores=False)
    check_against_oracle(LONG, inp, gpu)


@pytest.mark.parametrize("use_hist", [True, False])
def test_long_context_integer_ties_across_chunks(use_hist):
    cfg = LONG.with_(L=300, K=9000)
    inp, gpu, _ = run_case(cfg, seed=24, family="g1", bridge=0, code_dist="zipf", scores=False, use_hist=use_hist)
    check_against_oracle(cfg, inp, gpu, bridge=0)


@pytest.mark.parametrize("n_ctx", [70001, 65541, 33000])
def test_long_context_stream_select(n_ctx):
    # hist given and n_max % 16 == 0: one streaming CTA per pair (8192-token rounds, ragged
    # first / last round, window end inside a round)
    inp, gpu, _ = run_case(LONG, seed=25 + n_ctx % 7, scores=False, n_max=70016, n_ctx=n_ctx)
    check_against_oracle(LONG, inp, gpu, n_ctx=n_ctx)


def test_long_context_stream_integer_ties():
    # ties spread over many rounds: the quota m is carried across rounds in token order
    cfg = LONG.with_(L=300, K=9000)
    inp, gpu, _ = run_case(cfg, seed=26, family="g1", bridge=0, code_dist="zipf", scores=False, n_max=70016)
    check_against_oracle(cfg, inp, gpu, bridge=0)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("lut_engine", [1, 2])
def test_gqa_group_sizes(G, lut_engine):
    cfg = Config("gqa", B=2, Hq=2 * G, Hkv=2, d=128, N=3000, L=512, K=180)
    inp, gpu, _ = run_case(cfg, seed=30 + G, lut_engine=lut_engine)
    check_against_oracle(cfg, inp, gpu)


@pytest.mark.parametrize("lut_engine", [1, 2])
def test_group_sum(lut_engine):
    cfg = Config("gsum", B=2, Hq=8, Hkv=2, d=128, N=5000, L=512, K=300)
    inp, gpu, _ = run_case(cfg, seed=41, family="g1", bridge=0, group_reduce=O.GROUP_SUM, lut_engine=lut_engine)
    check_against_oracle(cfg, inp, gpu, bridge=0, group_reduce=O.GROUP_SUM)


@pytest.mark.parametrize("n_ctx,k", [(1, 5), (7, 5), (64, 5), (65, 5), (66, 5), (68, 5), (69, 1), (70, 100),
                                     (1000, 0), (1000, 932), (1000, 10_000), (4093, 1)])
def test_degenerate_sizes(n_ctx, k):
    cfg = Config("deg", B=1, Hq=4, Hkv=1, d=128, N=n_ctx, L=64, K=k)
    inp, gpu, _ = run_case(cfg.with_(), seed=50 + n_ctx, n_ctx=n_ctx)
    check_against_oracle(cfg, inp, gpu, n_ctx=n_ctx)


def test_window_covers_context_equals_rope():
    cfg = Config("win", B=1, Hq=4, Hkv=1, d=128, N=60, L=64, K=5)
    inp, gpu, _ = run_case(cfg, seed=61)
    check_against_oracle(cfg, inp, gpu)


def test_hist_and_no_hist_bitwise_equal_and_deterministic():
    cfg = SMALL
    inp1, g1, _ = run_case(cfg, seed=71, use_hist=True, scores=False)
    inp2, g2, _ = run_case(cfg, seed=71, use_hist=False, scores=False)
    _, g3, _ = run_case(cfg, seed=71, use_hist=True, scores=False)
    np.testing.assert_array_equal(g1["sel"], g2["sel"])
    assert np.array_equal(g1["out"].view(np.uint32), g2["out"].view(np.uint32))
    assert np.array_equal(g1["out"].view(np.uint32), g3["out"].view(np.uint32))


def test_workspace_returns_to_zero_state_for_counters():
    # calling twice with the same workspace gives identical results (counters reset by the kernels)
    cfg = SMALL
    inp = make_inputs(cfg, 81, device="cpu", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(topk=cfg.K)
    shape = A.make_shape(cfg.B, cfg.Hq, cfg.Hkv, 128, cfg.L, inp["n_max"])
    ws = torch.zeros(A.a2ats_decode_workspace_bytes(shape, params), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(3):
        out = torch.empty((cfg.B, cfg.Hq, 128), device="cuda")
        A.a2ats_decode_step(shape, params, cfg.N, dev["q"], dev["k_cache"], dev["v_cache"], dev["codes"],
                            dev["codebook"], None, out, None, None, ws)
        outs.append(out.cpu())
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


def test_needle_attention():
    cfg = Config("needle", B=2, Hq=8, Hkv=2, d=128, N=8000, L=512, K=480)
    inp, gpu, _ = run_case(cfg, seed=91, family="needle")
    check_against_oracle(cfg, inp, gpu)


def test_lossless_codebook_exact_scores():
    # every key its own codeword: u^ equals the exact bridge score q~ . k_t (BJ pin), on the GPU
    cfg = Config("lossless", B=1, Hq=1, Hkv=1, d=128, N=1024, L=1024, K=100)
    inp = make_inputs(cfg, 101, device="cpu", with_h=False)
    inp["codebook"] = inp["k_cache"][0, :, :cfg.L].clone()
    inp["codes"] = torch.arange(cfg.N, dtype=torch.int32).view(1, 1, -1).to(torch.uint16)
    inp["codes"] = torch.nn.functional.pad(inp["codes"].to(torch.int32), (0, inp["n_max"] - cfg.N)).to(torch.uint16)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(topk=cfg.K)
    shape = A.make_shape(1, 1, 1, 128, cfg.L, inp["n_max"])
    ws = torch.zeros(A.a2ats_decode_workspace_bytes(shape, params), dtype=torch.uint8, device="cuda")
    out = torch.empty((1, 1, 128), device="cuda")
    sc = torch.empty((1, 1, cfg.N), device="cuda")
    A.a2ats_decode_step(shape, params, cfg.N, dev["q"], dev["k_cache"], dev["v_cache"], dev["codes"],
                        dev["codebook"], None, out, None, sc, ws)
    qrot = O.wrope_query(f64(inp["q"][0, 0]), 2048, O.inv_freq(128))
    exact = f64(inp["k_cache"][0, 0, :cfg.N]) @ qrot
    assert row_rel_max(sc.cpu().numpy()[0, 0], exact) <= SCORE_RTOL


# ------------------------------------------------------------------ encoding (a0)
@pytest.mark.parametrize("with_h", [True, False])
def test_build_codes_matches_oracle(with_h):
    cfg = Config("enc", B=3, Hq=8, Hkv=2, d=128, N=700, L=384, K=10)
    inp = make_inputs(cfg, 111, device="cpu", with_h=True)
    H = inp["H"] if with_h else None
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], None if H is None else dev["H"])
    dec.encode(dev["k_cache"], 0, 300)
    dec.encode(dev["k_cache"], 300, cfg.N)
    torch.cuda.synchronize()
    got = codes_np(dec.codes)
    C = f64(inp["codebook"])
    for b in range(cfg.B):
        for h in range(cfg.Hkv):
            keys = f64(inp["k_cache"][b, h, :cfg.N])
            ref = O.qavq_encode(keys, C[h], None if H is None else f64(H[h]))
            np.testing.assert_array_equal(got[b, h, :cfg.N], ref)
            np.testing.assert_array_equal(dec.hist[b, h].cpu().numpy(), np.bincount(ref, minlength=cfg.L))
    # with keys drawn around codewords, the codes recover the generating assignment
    if not with_h:
        np.testing.assert_array_equal(got[:, :, :cfg.N], codes_np(inp["z"])[:, :, :cfg.N])


@pytest.mark.parametrize("B,T,steps", [(3, 1, 4), (100, 2, 2), (130, 1, 2), (16, 17, 1)])
def test_build_codes_decode_regime(B, T, steps):
    """Few keys per head (the decode step; B*T <= 256 runs the codeword-major
    encoder, 16*17 = 272 the bulk one): codes and running histogram vs the oracle,
    L = 400 (ragged last codeword tile).  H gets a large antisymmetric part, which
    leaves (k-c)H(k-c)^T unchanged (x A x^T = 0), so the codes must not move."""
    cfg = Config("encd", B=B, Hq=2, Hkv=2, d=128, N=64, L=400, K=10)
    inp = make_inputs(cfg, 141 + B, device="cpu", with_h=True)
    H = inp["H"]
    g = torch.Generator().manual_seed(5)
    R = torch.randn(H.shape, generator=g, dtype=torch.float32) * H.abs().max()
    H_asym = H + (R - R.transpose(1, 2))
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], H_asym.cuda())
    t0 = 5
    for s in range(steps):
        dec.encode(dev["k_cache"], t0 + s * T, t0 + (s + 1) * T)
    torch.cuda.synchronize()
    t1 = t0 + steps * T
    got = codes_np(dec.codes)
    C = f64(inp["codebook"])
    for b in range(cfg.B):
        for h in range(cfg.Hkv):
            ref = O.qavq_encode(f64(inp["k_cache"][b, h, t0:t1]), C[h], f64(H[h]))
            np.testing.assert_array_equal(got[b, h, t0:t1], ref)
            np.testing.assert_array_equal(dec.hist[b, h].cpu().numpy(), np.bincount(ref, minlength=cfg.L))
    assert (got[:, :, :t0] == 0).all() and (got[:, :, t1:] == 0).all()  # only [t_begin, t_end) written
    # the workspace is left zeroed (reusable): encode again into a fresh array, same result
    again = torch.zeros_like(dec.codes)
    dec.encode(dev["k_cache"], t0, t1, update_hist=False, codes=again)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(codes_np(again)[:, :, t0:t1], got[:, :, t0:t1])


def test_build_codes_keys_equal_codewords_and_ties():
    cfg = Config("enc2", B=1, Hq=1, Hkv=1, d=128, N=256, L=128, K=10)
    inp = make_inputs(cfg, 121, device="cpu", with_h=True, family="g1")
    C = inp["codebook"].clone()
    C[0, 100] = C[0, 3]              # duplicate codeword: lowest index wins
    keys = torch.zeros((1, 1, inp["n_max"], 128), dtype=torch.bfloat16)
    keys[0, 0, :128] = C[0]
    dec = A.Decoder(1, 1, 1, cfg.L, inp["n_max"], C.cuda(), inp["H"].cuda())
    dec.encode(keys.cuda(), 0, 128)
    got = codes_np(dec.codes)[0, 0, :128]
    want = np.arange(128)
    want[100] = 3
    np.testing.assert_array_equal(got, want)


# ------------------------------------------------------------------ host-mapped K/V (offload gather, C3 mirror)
def test_host_mapped_kv():
    cfg = Config("host", B=2, Hq=8, Hkv=2, d=128, N=9000, L=512, K=540)
    inp = make_inputs(cfg, 131, device="cpu", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    redraw_for_gap(inp, cfg, cfg.N, 131)
    kh = inp["k_cache"].pin_memory()
    vh = inp["v_cache"].pin_memory()
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(topk=cfg.K, kv_location=A.A2ATS_KV_HOST_MAPPED)
    shape = A.make_shape(cfg.B, cfg.Hq, cfg.Hkv, 128, cfg.L, inp["n_max"])
    ws = torch.zeros(A.a2ats_decode_workspace_bytes(shape, params), dtype=torch.uint8, device="cuda")
    out = torch.empty((cfg.B, cfg.Hq, 128), device="cuda")
    sel = torch.empty((cfg.B, cfg.Hkv, cfg.K), dtype=torch.int32, device="cuda")
    A.a2ats_decode_step(shape, params, cfg.N, dev["q"], kh, vh, dev["codes"], dev["codebook"], None, out, sel, None,
                        ws, kv_host=True)
    torch.cuda.synchronize()
    gpu = dict(out=out.cpu().numpy(), sel=sel.cpu().numpy(), scores=None)
    check_against_oracle(cfg, inp, gpu)


# ------------------------------------------------------------------ full size (C2), sampled
def test_c2_full_size_sampled():
    cfg = CONFIGS["C2"]
    seed = 0xA2A75 + 2
    inp = make_inputs(cfg, seed, device="cuda", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    sample = [(0, 0), (3, 5), (7, 7), (15, 2), (9, 4), (12, 1)]
    host = dict(q=inp["q"].cpu(), codebook=inp["codebook"].cpu(), codes=inp["codes"].cpu())
    redraw_for_gap(host, cfg, cfg.N, seed, pairs=sample)
    inp["q"] = host["q"].cuda()
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"])
    dec.codes = inp["codes"]
    dec.hist = hist_of(inp["codes"], cfg.L, cfg.N)
    dec.set_topk(cfg.K)
    sel = torch.empty((cfg.B, cfg.Hkv, cfg.K), dtype=torch.int32, device="cuda")
    out = dec.step(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, sel_out=sel)
    torch.cuda.synchronize()
    s = sel.cpu().numpy()
    # properties at every pair: ascending, unique, inside the candidate range
    assert np.all(np.diff(s, axis=2) > 0)
    assert s.min() >= cfg.n_sink and s.max() < cfg.N - cfg.window
    small = dict(q=host["q"], codebook=host["codebook"], codes=host["codes"],
                 k_cache=_PairView(inp["k_cache"]), v_cache=_PairView(inp["v_cache"]))
    gpu = dict(out=out.cpu().numpy(), sel=s, scores=None)
    check_against_oracle(cfg, small, gpu, pairs=sample)


def test_c4_full_size_sampled():
    """BASELINE configs[3] on one GPU (B = 64, N = 131072, L = 4096, K = 7865): the long-context
    select (threshold kernel + persistent half-pair scan) and the attention in the launch
    configuration bench.py --config C4 times; every pair checked for validity, sampled pairs
    (both scan halves of different CTAs) against the oracle bit for bit / within 2e-3."""
    cfg = CONFIGS["C4"]
    seed = 0xA2A75 + 4
    inp = make_inputs(cfg, seed, device="cuda", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    del inp["z"]
    sample = [(0, 0), (17, 3), (40, 7), (63, 5)]
    host = dict(q=inp["q"].cpu(), codebook=inp["codebook"].cpu(), codes=inp["codes"].cpu())
    redraw_for_gap(host, cfg, cfg.N, seed, pairs=sample)
    inp["q"] = host["q"].cuda()
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"])
    dec.codes = inp["codes"]
    dec.hist = hist_of(inp["codes"], cfg.L, cfg.N)
    dec.set_topk(cfg.K)
    sel = torch.empty((cfg.B, cfg.Hkv, cfg.K), dtype=torch.int32, device="cuda")
    out = dec.step(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, sel_out=sel)
    sel2 = torch.empty_like(sel)
    dec.select(inp["q"], cfg.N, sel2)
    torch.cuda.synchronize()
    assert torch.equal(sel, sel2)
    s = sel.cpu().numpy()
    assert np.all(np.diff(s, axis=2) > 0)
    assert s.min() >= cfg.n_sink and s.max() < cfg.N - cfg.window
    small = dict(q=host["q"], codebook=host["codebook"], codes=host["codes"],
                 k_cache=_PairView(inp["k_cache"]), v_cache=_PairView(inp["v_cache"]))
    gpu = dict(out=out.cpu().numpy(), sel=s, scores=None)
    check_against_oracle(cfg, small, gpu, pairs=sample)


class _PairView:
    """Indexes [b, h] of a device tensor lazily so only sampled pairs cross to the host."""

    def __init__(self, t):
        self.t = t

    def __getitem__(self, idx):
        return self.t[idx].cpu()


# ------------------------------------------------------------------ fused append step (a0 + a1..a6)
@pytest.mark.parametrize("use_hist,K,big", [(True, 60, False), (False, 60, False), (True, 0, False),
                                             (True, 123, True)])
def test_decode_step_append_equals_two_calls(use_hist, K, big):
    """a2ats_decode_step_append(n) == a2ats_build_codes(n-1, n) + a2ats_decode_step(n):
    identical codes, histogram, selection and output (same arithmetic, fused launch).
    big: C2's shapes (B = 16, 32 q / 8 KV heads, L = 4096), where the prep kernel groups
    two code tiles per CTA to keep its roles resident in one wave."""
    cfg = Config("app", B=3, Hq=8, Hkv=2, d=128, N=900, L=384, K=K)
    if big:
        cfg = Config("appbig", B=16, Hq=32, Hkv=8, d=128, N=1500, L=4096, K=K)
    inp = make_inputs(cfg, 151, device="cpu", with_h=True)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(topk=cfg.K)
    mk = lambda: A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], dev["H"], params)
    d1, d2 = mk(), mk()
    for d in (d1, d2):
        d.encode(dev["k_cache"], 0, cfg.N - 1)
    ka = max(cfg.K, 1)
    sel1 = torch.full((cfg.B, cfg.Hkv, ka), -1, dtype=torch.int32, device="cuda")
    sel2 = sel1.clone()
    d1.encode(dev["k_cache"], cfg.N - 1, cfg.N, update_hist=use_hist)
    o1 = d1.step(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=sel1, use_hist=use_hist)
    o2 = d2.step_append(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=sel2, use_hist=use_hist)
    torch.cuda.synchronize()
    assert torch.equal(d1.codes, d2.codes)
    if use_hist:
        assert torch.equal(d1.hist, d2.hist)
        np.testing.assert_array_equal(d2.hist.cpu().numpy(), hist_of(d2.codes, cfg.L, cfg.N).cpu().numpy())
    if K:
        assert torch.equal(sel1, sel2)
    assert torch.equal(o1, o2)
    # and against the oracle's code for the new token
    C = f64(inp["codebook"])
    for b in range(cfg.B):
        for h in range(cfg.Hkv):
            ref = O.qavq_encode(f64(inp["k_cache"][b, h, cfg.N - 1:cfg.N]), C[h], f64(inp["H"][h]))
            assert codes_np(d2.codes)[b, h, cfg.N - 1] == ref[0]


def test_wide_batch_append_sampled():
    """512 (b, KV head) pairs (C4's B = 64) at a short context through a2ats_decode_step_append:
    the prep kernel's balancing (two LUT vector tiles, grouped code tiles, several window pairs
    per CTA) on sampled pairs vs the oracle, and the appended token's code."""
    cfg = Config("wide", B=64, Hq=32, Hkv=8, d=128, N=3000, L=4096, K=180)
    seed = 0xA2A75 + 9
    inp = make_inputs(cfg, seed, device="cuda", with_h=True)
    inp["codes"] = inp["z"].to(torch.uint16)
    sample = [(0, 0), (17, 3), (31, 7), (40, 1), (63, 6), (63, 0)]
    host = dict(q=inp["q"].cpu(), codebook=inp["codebook"].cpu(), codes=inp["codes"].cpu())
    redraw_for_gap(host, cfg, cfg.N, seed, pairs=sample)
    inp["q"] = host["q"].cuda()
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"])
    dec.codes = inp["codes"].clone()
    dec.hist = hist_of(inp["codes"], cfg.L, cfg.N - 1)
    dec.set_topk(cfg.K)
    sel = torch.empty((cfg.B, cfg.Hkv, cfg.K), dtype=torch.int32, device="cuda")
    out = dec.step_append(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, sel_out=sel)
    torch.cuda.synchronize()
    got_codes = codes_np(dec.codes)
    C = f64(host["codebook"])
    H = f64(inp["H"].cpu())
    for b, h in sample:
        ref = O.qavq_encode(f64(inp["k_cache"][b, h, cfg.N - 1:cfg.N].cpu()), C[h], H[h])
        assert got_codes[b, h, cfg.N - 1] == ref[0]
    np.testing.assert_array_equal(dec.hist.cpu().numpy(), hist_of(dec.codes, cfg.L, cfg.N).cpu().numpy())
    small = dict(q=host["q"], codebook=host["codebook"], codes=host["codes"],
                 k_cache=_PairView(inp["k_cache"]), v_cache=_PairView(inp["v_cache"]))
    gpu = dict(out=out.cpu().numpy(), sel=sel.cpu().numpy(), scores=None)
    check_against_oracle(cfg, small, gpu, pairs=sample)


@pytest.mark.parametrize("N,n_max,use_hist", [(3000, 3008, True), (3000, 3008, False), (70001, 70016, True),
                                             (70001, 70008, True)])
def test_select_topk_equals_decode_step(N, n_max, use_hist):
    """a2ats_select_topk (a1..a4 only) == the sel_out of a2ats_decode_step, bit for bit, on the
    fused, streaming and threshold + chunked-scan selection paths."""
    cfg = Config("seltk", B=2, Hq=8, Hkv=2, d=128, N=N, L=512, K=max(60, N // 16))
    inp = make_inputs(cfg, 161, device="cuda", with_h=False, n_max=n_max)
    codes = inp["z"].to(torch.uint16)
    params = A.Params(topk=cfg.K)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], None, params)
    dec.codes = codes
    dec.hist = hist_of(codes, cfg.L, N)
    S, cand, W = O.token_sets(N, cfg.window, cfg.n_sink)
    keff = min(cfg.K, cand.size)
    s1 = torch.full((cfg.B, cfg.Hkv, keff), -1, dtype=torch.int32, device="cuda")
    s2 = s1.clone()
    dec.step(inp["q"], inp["k_cache"], inp["v_cache"], N, sel_out=s1, use_hist=use_hist)
    dec.select(inp["q"], N, s2, use_hist=use_hist)
    torch.cuda.synchronize()
    assert torch.equal(s1, s2)
    assert int(s2.min()) >= 0


# ------------------------------------------------------------------ long contexts, many pairs
@pytest.mark.parametrize("family,code_dist,N,L", [("g1", "zipf", 40001, 300), ("g2", "uniform", 57345, 4096),
                                                  ("g1", "uniform", 90000, 1000)])
def test_select_many_pairs_long_context(family, code_dist, N, L):
    """a2ats_select_topk with hist on P = 512 pairs of long contexts: the persistent
    warp-specialized select (several units per CTA: forward / backward halves of a pair on
    different CTAs, double-buffered class tables, per-pair flags), every pair against the
    oracle's top-K (sort-based, Eq. 21 + reading Q12).  g1: integer scores, exact ties
    across both halves; g2: pairs whose distinct-level cut gap is <= 1e-3 (reading Q20) are
    checked for validity only.  Called twice on one workspace: identical results (the flags
    are re-armed)."""
    from synth.generators import _gen, make_codebook, make_codes, make_query
    B, Hq, Hkv = 64, 32, 8
    G = Hq // Hkv
    K = -(-6 * N // 100)
    bridge = 0 if family == "g1" else 2048
    n_max = (N + 16 + 63) // 64 * 64
    g = _gen(4242 + N, "cpu")
    C = make_codebook(Hkv, L, 128, family, g, "cpu")
    q = make_query(B, Hq, 128, family, g, "cpu")
    z = make_codes(B, Hkv, n_max, L, code_dist, g, "cpu")
    codes = z.to(torch.uint16).cuda()
    hist = hist_of(codes, L, N)
    params = A.Params(topk=K, bridge=bridge)
    shape = A.make_shape(B, Hq, Hkv, 128, L, n_max)
    ws = torch.zeros(A.a2ats_decode_workspace_bytes(shape, params), dtype=torch.uint8, device="cuda")
    S_, cand, W_ = O.token_sets(N, 64, 4)
    keff = min(K, cand.size)
    sel = torch.full((B, Hkv, keff), -1, dtype=torch.int32, device="cuda")
    A.a2ats_select_topk(shape, params, N, q.cuda(), codes, C.cuda(), hist, sel, ws)
    sel2 = torch.full_like(sel, -1)
    A.a2ats_select_topk(shape, params, N, q.cuda(), codes, C.cuda(), hist, sel2, ws)
    torch.cuda.synchronize()
    assert torch.equal(sel, sel2)
    got = sel.cpu().numpy()
    Cd, zc, freqs = f64(C), z.to(torch.int64).numpy(), O.inv_freq(128)
    checked = 0
    for b in range(B):
        for h in range(Hkv):
            qrot = O.wrope_query(f64(q[b, h * G:(h + 1) * G]), bridge, freqs)
            agg = O.group_aggregate(O.approx_scores(qrot, zc[b, h, :N], Cd[h]))
            ref = O.select_topk(agg, cand, K)
            s = got[b, h]
            if family == "g1" or cut_gap(agg, cand, K) > 1e-3:
                np.testing.assert_array_equal(s, ref, err_msg=f"top-K set of pair {(b, h)}")
                checked += 1
            else:  # valid: ascending candidates, the same multiset of levels above the cut
                assert np.all(np.diff(s) > 0) and np.all(np.isin(s, cand))
                np.testing.assert_allclose(np.sort(agg[s]), np.sort(agg[ref]), rtol=0, atol=2e-3)
    assert checked >= B * Hkv * 8 // 10


def test_stage_rows_and_host_output_equal_device_path():
    """a2ats_stage_rows (q and the new K/V rows from pinned host memory, one kernel) + a
    decode step whose output is mapped pinned host memory == the all-device path, bitwise."""
    cfg = Config("stage", B=4, Hq=16, Hkv=4, d=128, N=5000, L=512, K=300)
    inp = make_inputs(cfg, 77, device="cuda", with_h=True)
    n = cfg.N
    params = A.Params(topk=cfg.K)
    outs = []
    for staged in (False, True):
        kc, vc = inp["k_cache"].clone(), inp["v_cache"].clone()
        dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], params)
        dec.encode(kc, 0, n - 1)
        if staged:
            q_host = inp["q"].cpu().pin_memory()
            k_host = kc[:, :, n - 1].contiguous().cpu().pin_memory()
            v_host = vc[:, :, n - 1].contiguous().cpu().pin_memory()
            kc[:, :, n - 1] = 0
            vc[:, :, n - 1] = 0
            q_dev = torch.zeros_like(inp["q"])
            A.a2ats_stage_rows(dec.shape, n, q_host, k_host, v_host, q_dev, kc, vc)
            out = torch.full((cfg.B, cfg.Hq, 128), float("nan")).pin_memory()
            dec.step_append(q_dev, kc, vc, n, out=out)
            torch.cuda.synchronize()
            assert torch.equal(kc[:, :, n - 1].cpu(), k_host) and torch.equal(q_dev.cpu(), q_host)
            outs.append(out.clone())
        else:
            out = dec.step_append(inp["q"], kc, vc, n)
            torch.cuda.synchronize()
            outs.append(out.cpu())
    assert torch.equal(outs[0], outs[1])


def test_stage_rows_device_sources_and_errors():
    """a2ats_stage_rows with device sources, partial (NULL) sources, and its argument checks."""
    cfg = Config("stage2", B=2, Hq=4, Hkv=2, d=128, N=100, L=64, K=5)
    shape = A.make_shape(cfg.B, cfg.Hq, cfg.Hkv, 128, cfg.L, 128)
    kc = torch.zeros((2, 2, 128, 128), dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    q_src = torch.randn((2, 4, 128), device="cuda").to(torch.bfloat16)
    k_src = torch.randn((2, 2, 128), device="cuda").to(torch.bfloat16)
    q_dst = torch.zeros_like(q_src)
    A.a2ats_stage_rows(shape, 77, q_src, k_src, None, q_dst, kc, vc)
    torch.cuda.synchronize()
    assert torch.equal(q_dst, q_src) and torch.equal(kc[:, :, 76], k_src)
    assert int(vc.abs().sum()) == 0 and int(kc[:, :, :76].abs().sum()) == 0
    for bad_n in (0, 129):
        with pytest.raises(A.A2ATSError):
            A.a2ats_stage_rows(shape, bad_n, q_src, k_src, None, q_dst, kc, vc)
