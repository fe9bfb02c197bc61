"""GPU parity, round 2: the cases round 1 left open.

- approximate scores at the LUT tile widths the bench runs (NV = 64 at C2's B*G = 64;
  NV = 128 + the qprep kernel at C4's B*G = 256), 1e-4 row-relative (reading Q18);
- window sizes beyond the 64 precomputed window rows (the cs-table branch), other sink counts;
- an inv_freq override (theta = 5e5 with the llama3 frequency scaling) instead of theta = 1e4;
- exact top-K on every one of the 512 pairs of full-size C4 (gap-redrawn, reading Q20);
- a smaller topk on a reused workspace (zero-state counters stay in place);
- a2ats_stage_rows + the fused step, repeated with fresh host rows (no stale q / K read).
Every comparison is against the fp64 oracle (oracle/), element by element.
"""
import math

import numpy as np
import pytest
import torch

from helpers import GAP, OUT_RTOL, SCORE_RTOL, codes_np, cut_gap, f64, rel_l2, row_rel_max
from oracle import a2ats_oracle as O
from synth import CONFIGS, Config, make_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12665_b200 as A


def llama3_inv_freq(d=128, theta=5e5, factor=8.0, low=1.0, high=4.0, old_ctx=8192):
    """Llama-3.1 rotary frequencies (theta = 5e5, 'llama3' scaling), fp64 -- the case the
    inv_freq override of a2ats_params exists for (reading Q1)."""
    f = theta ** (-np.arange(0, d, 2, dtype=np.float64) / d)
    wavelen = 2 * math.pi / f
    lo_w, hi_w = old_ctx / low, old_ctx / high
    out = np.where(wavelen > lo_w, f / factor, f)
    mid = (wavelen <= lo_w) & (wavelen >= hi_w)
    smooth = (old_ctx / wavelen - low) / (high - low)
    return np.where(mid, (1 - smooth) * f / factor + smooth * f, out)


def hist_of(codes, L, n_ctx):
    c = codes[:, :, :n_ctx].to(torch.int64)
    h = torch.zeros((codes.shape[0], codes.shape[1], L), dtype=torch.int32, device=codes.device)
    h.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
    return h


def redraw(inp, cfg, n_ctx, seed, freqs, bridge, pairs=None):
    """Reading Q20: re-draw (seed + attempt) the queries of pairs whose distinct-level gap at
    the cut is <= 1e-3, with the test's rotation frequencies."""
    G = cfg.Hq // cfg.Hkv
    C = f64(inp["codebook"])
    codes = codes_np(inp["codes"])
    S, cand, W = O.token_sets(n_ctx, cfg.window, cfg.n_sink)
    for b, h in pairs or [(b, h) for b in range(cfg.B) for h in range(cfg.Hkv)]:
        for attempt in range(60):
            qrot = O.wrope_query(f64(inp["q"][b, h * G:(h + 1) * G]), bridge, freqs)
            agg = O.group_aggregate(O.approx_scores(qrot, codes[b, h, :n_ctx], C[h]))
            if cut_gap(agg, cand, cfg.K) > GAP:
                break
            g = torch.Generator(device="cpu").manual_seed(seed * 1000003 + (b * 131 + h) * 977 + attempt + 1)
            inp["q"][b, h * G:(h + 1) * G] = torch.randn((G, cfg.d), generator=g).to(torch.bfloat16)
        else:
            raise RuntimeError("no clean cut")


def run_and_check(cfg, seed, *, freqs=None, theta=1e4, scores=True, use_hist=True, pairs=None):
    freqs_o = O.inv_freq(cfg.d, theta) if freqs is None else np.asarray(freqs, dtype=np.float64)
    inp = make_inputs(cfg, seed, device="cpu", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    redraw(inp, cfg, cfg.N, seed, freqs_o, cfg.bridge)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K, rope_theta=theta,
                      inv_freq=None if freqs is None else tuple(float(x) for x in freqs))
    shape = A.make_shape(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.L, inp["n_max"])
    ws = torch.zeros(A.a2ats_decode_workspace_bytes(shape, params), dtype=torch.uint8, device="cuda")
    out = torch.full((cfg.B, cfg.Hq, cfg.d), float("nan"), device="cuda")
    S, cand, W = O.token_sets(cfg.N, cfg.window, cfg.n_sink)
    keff = min(cfg.K, cand.size)
    sel = torch.full((cfg.B, cfg.Hkv, max(keff, 1)), -1, dtype=torch.int32, device="cuda")
    sc = torch.empty((cfg.B, cfg.Hq, cfg.N), device="cuda") if scores else None
    hist = hist_of(dev["codes"], cfg.L, cfg.N) if use_hist else None
    A.a2ats_decode_step(shape, params, cfg.N, dev["q"], dev["k_cache"], dev["v_cache"], dev["codes"],
                        dev["codebook"], hist, out, sel, sc, ws)
    torch.cuda.synchronize()
    o, s = out.cpu().numpy(), sel.cpu().numpy()[:, :, :keff]
    scn = None if sc is None else sc.cpu().numpy()
    G = cfg.G
    C = f64(inp["codebook"])
    codes = codes_np(inp["codes"])
    worst = 0.0
    for b, h in pairs or [(b, h) for b in range(cfg.B) for h in range(cfg.Hkv)]:
        r = O.decode_step_pair(f64(inp["q"][b, h * G:(h + 1) * G]), f64(inp["k_cache"][b, h]),
                               f64(inp["v_cache"][b, h]), codes[b, h], C[h], cfg.N, window=cfg.window,
                               bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K, freqs=freqs_o)
        np.testing.assert_array_equal(s[b, h], r["sel"], err_msg=f"top-K set of pair {(b, h)}")
        for g in range(G):
            if scn is not None:
                e = row_rel_max(scn[b, h * G + g], r["scores"][g])
                worst = max(worst, e)
                assert e <= SCORE_RTOL, f"scores row {(b, h * G + g)}: {e}"
            e = rel_l2(o[b, h * G + g], r["out"][g])
            assert e <= OUT_RTOL, f"output row {(b, h * G + g)}: {e}"
    return worst


# ------------------------------------------------------------------ scores at production LUT tile widths
@pytest.mark.parametrize("B,note", [(16, "B*G = 64: one NV = 64 tile per head (C2's LUT tile)"),
                                    (64, "B*G = 256: two NV = 128 tiles + qprep_kernel (C4's LUT path)")])
def test_scores_at_wide_lut_tiles(B, note):
    cfg = Config("wide", B=B, Hq=32, Hkv=8, d=128, N=700, L=1024, K=60)
    pairs = [(b, h) for b in range(B) for h in range(8)][:: max(1, B // 8)]
    worst = run_and_check(cfg, 901 + B, pairs=pairs)
    assert worst <= SCORE_RTOL


@pytest.mark.parametrize("B,Hq,Hkv,L", [(10, 64, 8, 1000),   # G = 8, B*G = 80: one ragged tile, 125-row codeword tail
                                       (40, 16, 8, 512),    # G = 2, B*G = 80
                                       (20, 32, 8, 384),    # G = 4, B*G = 80, L not a multiple of 256
                                       (72, 8, 8, 256)])    # G = 1, B*G = 72
def test_scores_persistent_lut_group_sizes(B, Hq, Hkv, L):
    """The persistent LUT kernel (query tiles wider than 64 vectors, q~ tiles from qprep) for every
    group size and ragged vector / codeword tiles: scores at 1e-4, sets and outputs vs the oracle."""
    cfg = Config("plut", B=B, Hq=Hq, Hkv=Hkv, d=128, N=700, L=L, K=60)
    pairs = [(b, h) for b in range(B) for h in range(Hkv)][::max(1, B * Hkv // 12)]
    worst = run_and_check(cfg, 950 + B + Hq, pairs=pairs)
    assert worst <= SCORE_RTOL


# ------------------------------------------------------------------ window / sinks / frequencies
@pytest.mark.parametrize("window,n_sink", [(96, 4), (128, 0), (100, 7), (65, 1)])
def test_window_beyond_precomputed_rows(window, n_sink):
    """window > 64: rows past the 64 precomputed window logits take the cs-table branch of
    the attention kernel (Eq. 11 with relative positions up to w - 1)."""
    cfg = Config("win", B=2, Hq=8, Hkv=2, d=128, N=3000, L=256, K=200, window=window, n_sink=n_sink)
    run_and_check(cfg, 1000 + window + n_sink)


@pytest.mark.parametrize("window", [64, 128])
def test_window_long_context_select(window):
    """The long-context select computes the window logits in its threshold kernel: window 128
    exercises rows past its 64 precomputed ones there too (N spans several code chunks)."""
    cfg = Config("winL", B=1, Hq=4, Hkv=1, d=128, N=70001, L=512, K=4200, window=window)
    run_and_check(cfg, 1700 + window, scores=False)


def test_inv_freq_override_llama3():
    """a2ats_params.inv_freq = Llama-3.1's scaled frequencies (theta 5e5, llama3 scaling): the
    bridge rotation, the window table and the window logits all follow the override."""
    cfg = Config("freq", B=2, Hq=8, Hkv=2, d=128, N=2500, L=256, K=150)
    run_and_check(cfg, 77, freqs=llama3_inv_freq())


def test_rope_theta_500k():
    cfg = Config("theta", B=2, Hq=8, Hkv=2, d=128, N=2500, L=256, K=150, window=80)
    run_and_check(cfg, 78, theta=5e5)


def test_inv_freq_length_checked():
    with pytest.raises(ValueError):
        A.Params(topk=3, inv_freq=(1.0, 0.5)).c()


# ------------------------------------------------------------------ full C4: every pair bit-exact
def test_c4_all_pairs_exact_topk():
    """BASELINE configs[3] shapes (B = 64, N = 131072, L = 4096, K = 7865): a2ats_select_topk in
    the bench's launch configuration (threshold kernel + persistent half-pair scan), every one
    of the 512 (b, KV head) pairs compared with the oracle's top-K bit for bit."""
    cfg = CONFIGS["C4"]
    seed = 0xA2A75 + 40
    g = torch.Generator(device="cuda").manual_seed(seed)
    n_max = cfg.n_max()
    C = torch.randn((cfg.Hkv, cfg.L, cfg.d), generator=g, device="cuda").to(torch.bfloat16)
    q = torch.randn((cfg.B, cfg.Hq, cfg.d), generator=g, device="cuda").to(torch.bfloat16)
    codes = torch.randint(0, cfg.L, (cfg.B, cfg.Hkv, n_max), generator=g, device="cuda").to(torch.int32)
    host = dict(q=q.cpu(), codebook=C.cpu(), codes=codes.cpu())
    freqs = O.inv_freq(cfg.d)
    redraw(host, cfg, cfg.N, seed, freqs, cfg.bridge)
    q = host["q"].cuda()
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, n_max, C)
    dec.codes = codes.to(torch.uint16)
    dec.hist = hist_of(dec.codes, cfg.L, cfg.N)
    dec.set_topk(cfg.K)
    sel = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
    dec.select(q, cfg.N, sel)
    torch.cuda.synchronize()
    s = sel.cpu().numpy()
    Cn = f64(host["codebook"])
    cn = host["codes"].numpy()
    S, cand, W = O.token_sets(cfg.N, cfg.window, cfg.n_sink)
    G = cfg.G
    for b in range(cfg.B):
        for h in range(cfg.Hkv):
            qrot = O.wrope_query(f64(host["q"][b, h * G:(h + 1) * G]), cfg.bridge, freqs)
            agg = O.group_aggregate(O.approx_scores(qrot, cn[b, h, :cfg.N], Cn[h]))
            np.testing.assert_array_equal(s[b, h], O.select_topk(agg, cand, cfg.K), err_msg=f"pair {(b, h)}")


# ------------------------------------------------------------------ workspace reuse
def test_smaller_topk_on_reused_workspace():
    """The zero-on-entry counters (attention split counters, encode slots) sit at shape-only
    offsets: a decreasing topk on the same workspace keeps the output correct."""
    cfg = Config("reuse", B=2, Hq=8, Hkv=2, d=128, N=6000, L=256, K=400)
    inp = make_inputs(cfg, 515, device="cpu", with_h=True)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], dev["H"], A.Params(topk=cfg.K))
    dec.encode(dev["k_cache"], 0, cfg.N - 1)
    ref_dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], dev["H"], A.Params(topk=cfg.K))
    for k in (400, 150, 7, 0, 90):
        dec.set_topk(k)
        out = dec.step(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N - 1)
        ref_dec.codes, ref_dec.hist = dec.codes, dec.hist
        ref_dec.params.topk = k
        ref_dec.ws_dec = torch.zeros(A.a2ats_decode_workspace_bytes(ref_dec.shape, ref_dec.params),
                                     dtype=torch.uint8, device="cuda")  # fresh, zeroed workspace
        ref = ref_dec.step(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N - 1)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), f"topk {k}: reused workspace differs from a fresh one"


# ------------------------------------------------------------------ staged rows, repeated
def test_stage_rows_repeated_fresh_rows():
    """a2ats_stage_rows then the fused step, 12 steps in a row with fresh q / new K, V rows in
    pinned host memory each step: every step equals the all-device path bitwise (the step's
    first kernel must not read q or the new key before stage_rows has written them)."""
    cfg = Config("stage3", B=4, Hq=16, Hkv=4, d=128, N=3000, L=256, K=180)
    inp = make_inputs(cfg, 99, device="cuda", with_h=True)
    n0 = cfg.N - 12
    params = A.Params(topk=cfg.K)
    decs = {}
    caches = {}
    for staged in (False, True):
        kc, vc = inp["k_cache"].clone(), inp["v_cache"].clone()
        d = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], params)
        d.encode(kc, 0, n0)
        decs[staged], caches[staged] = d, (kc, vc)
    g = torch.Generator(device="cpu").manual_seed(5)
    q_dev = torch.zeros_like(inp["q"])
    for step in range(12):
        n = n0 + step + 1
        q_h = torch.randn(inp["q"].shape, generator=g).to(torch.bfloat16).pin_memory()
        k_h = torch.randn((cfg.B, cfg.Hkv, 128), generator=g).to(torch.bfloat16).pin_memory()
        v_h = torch.randn((cfg.B, cfg.Hkv, 128), generator=g).to(torch.bfloat16).pin_memory()
        kc, vc = caches[False]
        kc[:, :, n - 1] = k_h.cuda()
        vc[:, :, n - 1] = v_h.cuda()
        ref = decs[False].step_append(q_h.cuda(), kc, vc, n)
        kc, vc = caches[True]
        A.a2ats_stage_rows(decs[True].shape, n, q_h, k_h, v_h, q_dev, kc, vc)
        out = decs[True].step_append(q_dev, kc, vc, n)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), f"step {step}: staged path differs"
        assert torch.equal(decs[True].codes, decs[False].codes) and torch.equal(decs[True].hist, decs[False].hist)
