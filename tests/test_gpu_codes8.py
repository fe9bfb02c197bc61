"""GPU parity of uint8 codes (shape.code_bytes = 1, L <= 256): half the index memory
(aux-mem 1/256 instead of the paper's 2-byte 1/128).  The encoder writes uint8 codes equal
to the fp64 oracle's Eq. 14 argmin; the posting-list engine (build, select, decode step, fused
append step) reads them; its top-K sets and outputs match the oracle (gap-redrawn inputs, C1
shapes) and equal the uint16 run bit for bit; the code-scan entry points refuse uint8 codes."""
import numpy as np
import pytest
import torch

from helpers import OUT_RTOL, codes_np, f64, pair_oracle, redraw_for_gap, rel_l2
from oracle import a2ats_oracle as O
from synth import CONFIGS, Config, make_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12665_b200 as A


def test_build_codes_uint8_matches_oracle():
    cfg = Config("enc8", B=3, Hq=8, Hkv=2, d=128, N=900, L=256, K=10)
    inp = make_inputs(cfg, 211, device="cpu", with_h=True)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], dev["H"], code_bytes=1)
    assert dec.codes.dtype == torch.uint8
    dec.encode(dev["k_cache"], 0, 5)          # decode regime (few keys per head)
    dec.encode(dev["k_cache"], 5, cfg.N)      # bulk regime
    torch.cuda.synchronize()
    got = codes_np(dec.codes)
    C = f64(inp["codebook"])
    for b in range(cfg.B):
        for h in range(cfg.Hkv):
            ref = O.qavq_encode(f64(inp["k_cache"][b, h, :cfg.N]), C[h], f64(inp["H"][h]))
            np.testing.assert_array_equal(got[b, h, :cfg.N], ref)
            np.testing.assert_array_equal(dec.hist[b, h].cpu().numpy(), np.bincount(ref, minlength=cfg.L))
    assert int(got[:, :, cfg.N:].max()) == 0  # nothing written past t_end


@pytest.mark.parametrize("frac", [1.0, 0.95, 0.3])
def test_postings_step_uint8_matches_oracle(frac):
    cfg = CONFIGS["C1"].with_(B=2, Hkv=2, Hq=8)
    inp = make_inputs(cfg, 212, device="cpu", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    redraw_for_gap(inp, cfg, cfg.N, 212)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    res = {}
    for cb in (2, 1):
        params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K)
        dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], None, params, code_bytes=cb)
        dec.codes = dev["codes"].to(torch.uint8) if cb == 1 else dev["codes"]
        c = dev["codes"][:, :, :cfg.N].to(torch.int64)
        dec.hist = torch.zeros((cfg.B, cfg.Hkv, cfg.L), dtype=torch.int32, device="cuda")
        dec.hist.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
        dec.build_postings(int(cfg.N * frac))
        sel = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
        out = dec.step_postings(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=sel)
        torch.cuda.synchronize()
        res[cb] = (sel.cpu().numpy(), out.cpu().numpy())
    np.testing.assert_array_equal(res[1][0], res[2][0])
    assert np.array_equal(res[1][1].view(np.uint32), res[2][1].view(np.uint32))
    G = cfg.Hq // cfg.Hkv
    codes = codes_np(inp["codes"])
    C = f64(inp["codebook"])
    for b in range(cfg.B):
        for h in range(cfg.Hkv):
            r = pair_oracle(f64(inp["q"][b, h * G:(h + 1) * G]), f64(inp["k_cache"][b, h]), f64(inp["v_cache"][b, h]),
                            codes[b, h], C[h], cfg.N, cfg)
            np.testing.assert_array_equal(np.sort(res[1][0][b, h]), r["sel"])
            for g in range(G):
                assert rel_l2(res[1][1][b, h * G + g], r["out"][g]) <= OUT_RTOL


def test_append_postings_uint8_equals_uint16():
    cfg = Config("app8", B=2, Hq=8, Hkv=2, d=128, N=6000, L=256, K=400)
    steps = 4
    inp = make_inputs(cfg, 213, device="cuda", with_h=True, n_max=cfg.n_max(extra=steps + 8))
    runs = {}
    for cb in (2, 1):
        params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K)
        dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], params, code_bytes=cb)
        n0 = cfg.N - steps
        dec.encode(inp["k_cache"], 0, n0)
        dec.build_postings(n0 - cfg.window - 100)
        sels, outs = [], []
        for s in range(steps):
            sel = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
            outs.append(dec.step_append_postings(inp["q"], inp["k_cache"], inp["v_cache"], n0 + s + 1,
                                                 sel_out=sel).clone())
            sels.append(sel)
        torch.cuda.synchronize()
        runs[cb] = (dec.codes.to(torch.int32), dec.hist.clone(), sels, outs)
    assert torch.equal(runs[1][0], runs[2][0]) and torch.equal(runs[1][1], runs[2][1])
    for s in range(steps):
        assert torch.equal(runs[1][2][s], runs[2][2][s])
        assert torch.equal(runs[1][3][s], runs[2][3][s])


def test_uint8_codes_refused_by_scan_engines_and_wide_codebooks():
    cfg = Config("ref8", B=1, Hq=4, Hkv=1, d=128, N=500, L=256, K=20)
    inp = make_inputs(cfg, 214, device="cuda", with_h=False)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], None,
                    A.Params(topk=cfg.K), code_bytes=1)
    with pytest.raises(Exception, match="UNSUPPORTED"):
        dec.step(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N)
    sel = torch.empty((1, 1, cfg.K), dtype=torch.int32, device="cuda")
    with pytest.raises(Exception, match="UNSUPPORTED"):
        dec.select(inp["q"], cfg.N, sel)
    with pytest.raises(Exception, match="UNSUPPORTED"):
        A.Decoder(1, 4, 1, 300, inp["n_max"], torch.zeros((1, 300, 128), dtype=torch.bfloat16, device="cuda"),
                  None, code_bytes=1)
