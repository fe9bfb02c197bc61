"""Deferred a0 (params.hist_lag: a new token's code is first read when it leaves the
window): with the newest `lag` tokens not encoded -- their codes garbage, hist covering
[0, N - lag) -- every selection engine returns the same top-K and the same output bit for bit as
with every token encoded (hist_lag = 0), which the other GPU tests pin to the fp64 oracle.  Plus
the batched-encode policy of the bench: a2ats_build_codes of the last window of tokens every
`window` steps reproduces the per-step fused append exactly."""
import numpy as np
import pytest
import torch

from synth import Config, make_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12665_b200 as A


def hist_of(codes, L, n):
    c = codes[:, :, :n].to(torch.int64)
    h = torch.zeros((codes.shape[0], codes.shape[1], L), dtype=torch.int32, device=codes.device)
    h.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
    return h


def run(cfg, inp, lag, engine, select_only=False):
    params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K, hist_lag=lag)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], None, params)
    z = inp["z"].to(torch.int64).clone()
    if lag:
        z[:, :, cfg.N - lag:cfg.N] = cfg.L - 1 - z[:, :, cfg.N - lag:cfg.N]  # not encoded yet: garbage
    codes = z.to(torch.uint16)
    dec.hist = hist_of(inp["z"].to(torch.uint16), cfg.L, cfg.N - lag)
    dec.codes = codes
    sel = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
    out = None
    if engine == "postings":
        dec.build_postings(cfg.N - cfg.window - 300)
        if select_only:
            dec.select_postings(inp["q"], cfg.N, sel)
        else:
            out = dec.step_postings(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, sel_out=sel)
    elif select_only:
        dec.select(inp["q"], cfg.N, sel, use_hist=engine != "nohist")
    else:
        out = dec.step(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, sel_out=sel, use_hist=engine != "nohist")
    torch.cuda.synchronize()
    return sel.cpu(), None if out is None else out.cpu()


@pytest.mark.parametrize("engine,N,L", [("scan", 9000, 512), ("scan", 70000, 512), ("nohist", 70000, 512),
                                        ("postings", 20000, 1024)])
@pytest.mark.parametrize("lag", [1, 37, 64])
def test_deferred_encode_identical(engine, N, L, lag):
    cfg = Config("lag", B=2, Hq=8, Hkv=2, d=128, N=N, L=L, K=int(np.ceil(0.06 * N)))
    inp = make_inputs(cfg, 300 + lag, device="cuda", with_h=False)
    s0, o0 = run(cfg, inp, 0, engine)
    s1, o1 = run(cfg, inp, lag, engine)
    assert torch.equal(s0, s1)
    assert torch.equal(o0, o1)
    s2, _ = run(cfg, inp, lag, engine, select_only=True)
    assert torch.equal(torch.sort(s0, dim=2).values, torch.sort(s2, dim=2).values)


def test_hist_lag_argument_checks():
    cfg = Config("lagc", B=1, Hq=4, Hkv=1, d=128, N=2000, L=256, K=50)
    inp = make_inputs(cfg, 310, device="cuda", with_h=False)
    with pytest.raises(Exception):
        run(cfg, inp, 65, "scan")  # more than the window
    params = A.Params(topk=cfg.K, hist_lag=3)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], None, params)
    with pytest.raises(Exception):  # the fused append encodes token N - 1 itself: no lag
        dec.step_append(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N)


def test_batched_encode_policy_equals_fused_append():
    """Every `window` steps encode the newest tokens in one a2ats_build_codes call, steps in between
    with hist_lag = n - n_encoded: the same codes, histogram, selections and outputs as the per-step
    fused append (a2ats_decode_step_append_postings)."""
    cfg = Config("lagp", B=2, Hq=8, Hkv=2, d=128, N=12000, L=512, K=700)
    steps = 70
    inp = make_inputs(cfg, 311, device="cuda", with_h=True, n_max=cfg.n_max(extra=steps + 8))
    q, kc, vc = inp["q"], inp["k_cache"], inp["v_cache"]
    n0 = cfg.N - steps
    decs = []
    for lagged in (False, True):
        params = A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K)
        d = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], params)
        d.encode(kc, 0, n0)
        d.build_postings(n0 - cfg.window - 200)
        decs.append(d)
    fused, lagged = decs
    n_enc = n0
    for s in range(steps):
        n = n0 + s + 1
        s1 = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
        s2 = torch.full_like(s1, -1)
        o1 = fused.step_append_postings(q, kc, vc, n, sel_out=s1)
        if n - n_enc > cfg.window:  # the oldest unencoded token would leave the window: encode the batch
            lagged.encode(kc, n_enc, n - 1)
            n_enc = n - 1
        lagged.params.hist_lag = n - n_enc
        o2 = lagged.step_postings(q, kc, vc, n, sel_out=s2)
        torch.cuda.synchronize()
        assert torch.equal(s1, s2), s
        assert torch.equal(o1, o2), s
    lagged.encode(kc, n_enc, n0 + steps)
    torch.cuda.synchronize()
    assert torch.equal(fused.codes[:, :, :n0 + steps], lagged.codes[:, :, :n0 + steps])
    assert torch.equal(fused.hist, lagged.hist)


@pytest.mark.parametrize("engine", ["scan", "postings"])
def test_decoder_serving_loop_equals_fused_append(engine):
    """Decoder.start / decode (batched a0 every window, posting index rebuilt every few steps) over
    a run of decode steps == the fused append step of every step: the same codes, histogram and
    top-K sets; outputs equal up to the summation order of the rows (index order)."""
    cfg = Config("loop", B=2, Hq=8, Hkv=2, d=128, N=9000, L=512, K=540)
    steps = 150
    inp = make_inputs(cfg, 320, device="cuda", with_h=True, n_max=cfg.n_max(extra=steps + 8))
    q, kc, vc = inp["q"], inp["k_cache"], inp["v_cache"]
    n0 = cfg.N - steps
    mk = lambda: A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"],
                           A.Params(window=cfg.window, bridge=cfg.bridge, n_sink=cfg.n_sink, topk=cfg.K))
    ref, dut = mk(), mk()
    ref.encode(kc, 0, n0)
    dut.start(kc, n0, engine=engine, rebuild_every=40)
    for s in range(steps):
        n = n0 + s + 1
        s1 = torch.full((cfg.B, cfg.Hkv, cfg.K), -1, dtype=torch.int32, device="cuda")
        s2 = torch.full_like(s1, -1)
        o1 = ref.step_append(q, kc, vc, n, sel_out=s1)
        o2 = dut.decode(q, kc, vc, n, sel_out=s2)
        torch.cuda.synchronize()
        assert torch.equal(s1, torch.sort(s2, dim=2).values), s
        rel = ((o1 - o2).norm(dim=2) / o1.norm(dim=2)).max().item()
        assert rel <= 1e-5, (s, rel)
    dut.encode(kc, dut._n_enc, n0 + steps)
    torch.cuda.synchronize()
    assert torch.equal(ref.codes[:, :, :n0 + steps], dut.codes[:, :, :n0 + steps])
    assert torch.equal(ref.hist, dut.hist)
