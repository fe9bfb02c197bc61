"""GPU parity of the standard-RoPE ablation mode (params.rope_mode = A2ATS_ROPE_STANDARD; the
"Baseline" / "QAVQ" configurations of P:419-427) against the oracle's decode_step_pair_standard:
the cache holds post-PE keys, q~ = q R_{N-1}, every selected row gets the standard logit.  Top-K
sets bit-exact (queries re-drawn until the distinct-level gap at the cut exceeds 1e-3, reading
Q20), outputs within 2e-3; one-chunk, long-context and posting-list engines, append step."""
import numpy as np
import pytest
import torch

from helpers import GAP, OUT_RTOL, codes_np, cut_gap, f64, rel_l2
from oracle import a2ats_oracle as O
from synth import Config, make_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12665_b200 as A

STD = 1  # A2ATS_ROPE_STANDARD


def redraw(inp, cfg, seed, pairs):
    G = cfg.Hq // cfg.Hkv
    C = f64(inp["codebook"])
    codes = codes_np(inp["codes"])
    S, cand, W = O.token_sets(cfg.N, cfg.window, cfg.n_sink)
    for b, h in pairs:
        for attempt in range(40):
            qr = O.rope_rotate(f64(inp["q"][b, h * G:(h + 1) * G]), cfg.N - 1, O.inv_freq(cfg.d))
            agg = O.group_aggregate(O.approx_scores(qr, codes[b, h, :cfg.N], C[h]))
            if cut_gap(agg, cand, cfg.K) > GAP:
                break
            g = torch.Generator().manual_seed(seed * 1000 + b * 37 + h * 5 + attempt)
            inp["q"][b, h * G:(h + 1) * G] = torch.randn((G, cfg.d), generator=g).to(torch.bfloat16)


@pytest.mark.parametrize("engine,N,L", [("scan", 3000, 256), ("scan", 70001, 512), ("postings", 12000, 512)])
def test_standard_rope_matches_oracle(engine, N, L):
    cfg = Config("std", B=2, Hq=8, Hkv=2, d=128, N=N, L=L, K=int(np.ceil(0.06 * N)))
    inp = make_inputs(cfg, 400 + N % 97, device="cpu", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    pairs = [(0, 0), (1, 1)] if N > 10000 else [(b, h) for b in range(cfg.B) for h in range(cfg.Hkv)]
    redraw(inp, cfg, 400 + N % 97, pairs)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K, rope_mode=STD)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], None, params)
    dec.codes = dev["codes"]
    c = dev["codes"][:, :, :cfg.N].to(torch.int64)
    dec.hist = torch.zeros((cfg.B, cfg.Hkv, cfg.L), dtype=torch.int32, device="cuda")
    dec.hist.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
    sel = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
    if engine == "postings":
        dec.build_postings(cfg.N - cfg.window - 300)
        out = dec.step_postings(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=sel)
    else:
        out = dec.step(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=sel)
    torch.cuda.synchronize()
    sel, out = sel.cpu().numpy(), out.cpu().numpy()
    G = cfg.Hq // cfg.Hkv
    C = f64(inp["codebook"])
    codes = codes_np(inp["codes"])
    for b, h in pairs:
        r = O.decode_step_pair_standard(f64(inp["q"][b, h * G:(h + 1) * G]), f64(inp["k_cache"][b, h]),
                                        f64(inp["v_cache"][b, h]), codes[b, h], C[h], cfg.N, window=cfg.window,
                                        n_sink=cfg.n_sink, topk=cfg.K)
        np.testing.assert_array_equal(np.sort(sel[b, h]), r["sel"], err_msg=f"pair {(b, h)}")
        for g in range(G):
            e = rel_l2(out[b, h * G + g], r["out"][g])
            assert e <= OUT_RTOL, f"row {(b, h * G + g)} rel L2 {e}"


def test_standard_rope_differs_from_wrope_and_append_matches():
    """The mode changes the result (window rows and the query rotation differ from WRoPE), and the
    fused append step (a0 for the new token) equals build_codes + the step."""
    cfg = Config("std2", B=2, Hq=8, Hkv=2, d=128, N=3000, L=256, K=180)
    inp = make_inputs(cfg, 410, device="cuda", with_h=True)
    outs = []
    for mode, append in ((0, False), (STD, False), (STD, True)):
        params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K, rope_mode=mode)
        dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], params)
        if append:
            dec.encode(inp["k_cache"], 0, cfg.N - 1)
            o = dec.step_append(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N)
        else:
            dec.encode(inp["k_cache"], 0, cfg.N)
            o = dec.step(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N)
        torch.cuda.synchronize()
        outs.append(o.clone())
    assert (outs[0] - outs[1]).abs().max() > 1e-3
    assert torch.equal(outs[1], outs[2])
