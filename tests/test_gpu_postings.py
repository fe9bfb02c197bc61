"""GPU parity of the posting-list (inverted-index) selection engine:
a2ats_select_topk_postings / a2ats_decode_step_postings produce the same top-K SETS as the
code-scan engine -- which the other GPU tests pin to the fp64 oracle -- and match the oracle
directly on sampled pairs; the attention output equals the scan engine's up to the summation
order of the rows (the list path emits the set in index order, not ascending); with the index
covering all (bitmap path: window tokens in the index), part or none of the candidates
(tokens not yet indexed are classified from their codes), integer ties across codes, Zipf
code usage and long contexts.  The index itself (a2ats_postings_build) is checked exactly
against a stable sort of the tokens by code."""
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
    a1, a2 = s1.cpu().numpy(), s2.cpu().numpy()
    np.testing.assert_array_equal(np.sort(a2, axis=2), a1)  # same sets (scan engine: ascending)
    if attend:
        d = (o1 - o2).norm(dim=2) / o1.norm(dim=2)
        assert float(d.max()) <= 1e-5, float(d.max())
    return np.sort(a2, axis=2), None if o2 is None else o2.cpu().numpy()


@pytest.mark.parametrize("frac", [1.0, 0.99, 0.6, 0.0])
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


@pytest.mark.parametrize("N,L,frac", [(70001, 4096, 1.0), (131072, 4096, 0.999), (131072, 4096, 0.99),
                                      (131072, 4096, 0.9), (40000, 1000, 0.5)])
def test_postings_long_contexts_select_only(N, L, frac):
    cfg = Config("postl", B=4, Hq=32, Hkv=8, d=128, N=N, L=L, K=int(np.ceil(0.06 * N)))
    g = torch.Generator(device="cuda").manual_seed(N)
    n_max = cfg.n_max()
    inp = dict(codebook=torch.randn((8, L, 128), generator=g, device="cuda").to(torch.bfloat16),
               q=torch.randn((4, 32, 128), generator=g, device="cuda").to(torch.bfloat16),
               codes=torch.randint(0, L, (4, 8, n_max), generator=g, device="cuda").to(torch.uint16), n_max=n_max)
    both(cfg, inp, frac, attend=False)


def test_postings_zipf_list_path():
    """Zipf code usage (long lists, several tied codes under integer ties), index short of the window."""
    cfg = Config("postz2", B=2, Hq=8, Hkv=2, d=128, N=12000, L=300, K=3000, bridge=0)
    inp = make_inputs(cfg, 63, device="cpu", family="g1", code_dist="zipf", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    both(cfg, inp, 0.95)


def test_postings_index_is_stable_sort_by_code():
    """post_off / post_tok == the stable sort of tokens [0, n) by code (lists ascending), exactly."""
    B, Hkv, L, n_max, n = 3, 2, 700, 5056, 5000
    g = torch.Generator(device="cuda").manual_seed(7)
    codes = torch.randint(0, L, (B, Hkv, n_max), generator=g, device="cuda").to(torch.uint16)
    codes[0, 0, :2000] = 5                      # one very long list
    shape = A.make_shape(B, 2 * Hkv, Hkv, 128, L, n_max)
    post = torch.zeros(A.binding.a2ats_postings_bytes(shape), dtype=torch.uint8, device="cuda")
    A.binding.a2ats_postings_build(shape, codes, n, post)
    torch.cuda.synchronize()
    P = B * Hkv
    LP = (L + 4) // 4 * 4                       # a2ats.h: offset rows of L + 1 padded to 16 B
    t0 = (P * LP * 4 + 255) // 256 * 256        # offsets, then tokens (256-B aligned)
    off = post[:P * LP * 4].view(torch.int32).view(P, LP)[:, :L + 1].cpu().numpy()
    tok = post[t0:t0 + P * n_max * 4].view(torch.int32).view(P, n_max).cpu().numpy()
    c = codes.view(P, n_max)[:, :n].cpu().numpy().astype(np.int64)
    for p in range(P):
        order = np.argsort(c[p], kind="stable")
        np.testing.assert_array_equal(tok[p, :n], order)
        np.testing.assert_array_equal(off[p], np.concatenate([[0], np.cumsum(np.bincount(c[p], minlength=L))]))


def test_postings_list_path_deterministic():
    cfg = Config("postd", B=2, Hq=8, Hkv=2, d=128, N=20000, L=1024, K=1200)
    inp = make_inputs(cfg, 64, device="cpu", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], None, params)
    dec.codes = dev["codes"]
    dec.hist = hist_of(dev["codes"], cfg.L, cfg.N)
    outs = []
    for _ in range(2):
        dec.build_postings(cfg.N - 500)
        s = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
        o = dec.step_postings(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=s)
        torch.cuda.synchronize()
        outs.append((s.clone(), o.clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_append_postings_steps_equal_append_scan():
    """a2ats_decode_step_append_postings over several decode steps (the index built once, the
    unindexed tail growing by one token per step, one rebuild half-way) == a2ats_decode_step_append
    (scan engine): the same new codes, the same running histogram, the same top-K sets, the
    same output up to the row summation order."""
    cfg = Config("posta", B=2, Hq=8, Hkv=2, d=128, N=20000, L=512, K=1200)
    steps = 6
    inp = make_inputs(cfg, 65, device="cuda", with_h=True, n_max=cfg.n_max(extra=steps + 8))
    q, kc, vc = inp["q"], inp["k_cache"], inp["v_cache"]
    params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K)
    d1 = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], params)
    d2 = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"],
                   A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K))
    n0 = cfg.N - steps
    d1.encode(kc, 0, n0)
    d2.encode(kc, 0, n0)
    d2.build_postings(n0 - cfg.window - 300)
    for s in range(steps):
        n = n0 + s + 1
        if s == steps // 2:
            d2.build_postings(n - 1 - cfg.window)  # the whole candidate range indexed
        s1 = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
        s2 = torch.full_like(s1, -1)
        o1 = d1.step_append(q, kc, vc, n, sel_out=s1)
        o2 = d2.step_append_postings(q, kc, vc, n, sel_out=s2)
        torch.cuda.synchronize()
        assert torch.equal(d1.codes[:, :, :n], d2.codes[:, :, :n])
        assert torch.equal(d1.hist, d2.hist)
        np.testing.assert_array_equal(np.sort(s2.cpu().numpy(), axis=2), s1.cpu().numpy())
        rel = (o1 - o2).norm(dim=2) / o1.norm(dim=2)
        assert float(rel.max()) <= 1e-5, float(rel.max())
    # the running histogram is the histogram of the final codes
    assert torch.equal(d2.hist, hist_of(d2.codes, cfg.L, n0 + steps))
