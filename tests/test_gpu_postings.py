"""GPU parity of the posting-list (inverted-index) selection engine:
a2ats_select_topk_postings / a2ats_decode_step_postings produce the same top-K sets (same
order) and the same output, bitwise, as the code-scan engine -- which the other GPU tests pin
to the fp64 oracle -- and match the oracle directly on sampled pairs; with the index covering
all, part or none of the candidates (tokens not yet indexed are classified from their codes),
integer ties across codes, Zipf code usage and long contexts."""
import numpy as np
import pytest
import torch

from helpers import codes_np, f64, pair_oracle, redraw_for_gap
from synth import Config, make_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12665_b200 as A


def hist_of(codes, L, n):
    c = codes[:, :, :n].to(torch.int64)
    h = torch.zeros((codes.shape[0], codes.shape[1], L), dtype=torch.int32, device=codes.device)
    h.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
    return h


def both(cfg, inp, n_post_frac, attend=True):
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], None, params)
    dec.codes = dev["codes"]
    dec.hist = hist_of(dev["codes"], cfg.L, cfg.N)
    n_post = int(cfg.N * n_post_frac)
    dec.build_postings(n_post)
    s1 = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
    s2 = torch.full_like(s1, -1)
    if attend:
        o1 = dec.step(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=s1)
        o2 = dec.step_postings(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=s2)
    else:
        dec.select(dev["q"], cfg.N, s1)
        dec.select_postings(dev["q"], cfg.N, s2)
        o1 = o2 = None
    torch.cuda.synchronize()
    assert torch.equal(s1, s2)
    if attend:
        assert torch.equal(o1, o2)
    return s2.cpu().numpy(), None if o2 is None else o2.cpu().numpy()


@pytest.mark.parametrize("frac", [1.0, 0.6, 0.0])
def test_postings_equal_scan_engine(frac):
    cfg = Config("post", B=2, Hq=8, Hkv=2, d=128, N=9000, L=512, K=600)
    inp = make_inputs(cfg, 61, device="cpu", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    redraw_for_gap(inp, cfg, cfg.N, 61)
    sel, out = both(cfg, inp, frac)
    G = cfg.G
    C = f64(inp["codebook"])
    codes = codes_np(inp["codes"])
    for b, h in [(0, 0), (1, 1)]:
        r = pair_oracle(f64(inp["q"][b, h * G:(h + 1) * G]), f64(inp["k_cache"][b, h]), f64(inp["v_cache"][b, h]),
                        codes[b, h], C[h], cfg.N, cfg)
        np.testing.assert_array_equal(sel[b, h], r["sel"])


def test_postings_integer_ties_zipf():
    cfg = Config("postz", B=2, Hq=8, Hkv=2, d=128, N=12000, L=300, K=3000, bridge=0)
    inp = make_inputs(cfg, 62, device="cpu", family="g1", code_dist="zipf", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    both(cfg, inp, 0.8)


@pytest.mark.parametrize("N,L,frac", [(70001, 4096, 1.0), (131072, 4096, 0.999), (40000, 1000, 0.5)])
def test_postings_long_contexts_select_only(N, L, frac):
    cfg = Config("postl", B=4, Hq=32, Hkv=8, d=128, N=N, L=L, K=int(np.ceil(0.06 * N)))
    g = torch.Generator(device="cuda").manual_seed(N)
    n_max = cfg.n_max()
    inp = dict(codebook=torch.randn((8, L, 128), generator=g, device="cuda").to(torch.bfloat16),
               q=torch.randn((4, 32, 128), generator=g, device="cuda").to(torch.bfloat16),
               codes=torch.randint(0, L, (4, 8, n_max), generator=g, device="cuda").to(torch.uint16), n_max=n_max)
    both(cfg, inp, frac, attend=False)
