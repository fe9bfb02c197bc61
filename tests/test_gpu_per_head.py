"""GPU parity of per-query-head selection (A2ATS_GROUP_PER_HEAD): every
query head selects its own top-K from its own LUT row and attends over its own Sel.  The oracle of
query head hq is the single-head oracle (G = 1) of that head on its KV head's codes, keys and
values.  Integer-exact inputs (g1 family, bridge 0) make every tie exact on both sides, so the
sets are compared bit for bit; outputs within the 2e-3 relative L2 of reading Q19.  Covers the
scan engines (one-chunk fused and long-context), the posting-list engine, select-only, the fused
append step (a0 once, then G sub-steps over the updated histogram), G in {2, 4, 8}."""
import numpy as np
import pytest
import torch

from helpers import OUT_RTOL, codes_np, f64, rel_l2
from oracle import a2ats_oracle as O
from synth import Config, make_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12665_b200 as A

PH = 2  # A2ATS_GROUP_PER_HEAD


def head_oracle(inp, cfg, b, hq, n_ctx, bridge):
    G = cfg.Hq // cfg.Hkv
    h = hq // G
    return O.decode_step_pair(f64(inp["q"][b, hq:hq + 1]), f64(inp["k_cache"][b, h]), f64(inp["v_cache"][b, h]),
                              codes_np(inp["codes"])[b, h], f64(inp["codebook"])[h], n_ctx, window=cfg.window,
                              bridge=bridge, n_sink=cfg.n_sink, topk=cfg.K)


def run(cfg, seed, *, postings=None, select_only=False, bridge=0, family="g1", code_dist="uniform"):
    inp = make_inputs(cfg, seed, device="cpu", family=family, code_dist=code_dist, with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(window=cfg.window, bridge=bridge, n_sink=cfg.n_sink, topk=cfg.K, group_reduce=PH)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], None, params)
    dec.codes = dev["codes"]
    c = dev["codes"][:, :, :cfg.N].to(torch.int64)
    dec.hist = torch.zeros((cfg.B, cfg.Hkv, cfg.L), dtype=torch.int32, device="cuda")
    dec.hist.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
    S, cand, W = O.token_sets(cfg.N, cfg.window, cfg.n_sink)
    keff = min(cfg.K, cand.size)
    sel = torch.full((cfg.B, cfg.Hq, max(keff, 1)), -1, dtype=torch.int32, device="cuda")
    out = None
    if postings is not None:
        dec.build_postings(int(cfg.N * postings))
        if select_only:
            dec.select_postings(dev["q"], cfg.N, sel)
        else:
            out = dec.step_postings(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=sel)
    elif select_only:
        dec.select(dev["q"], cfg.N, sel)
    else:
        out = dec.step(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=sel)
    torch.cuda.synchronize()
    return inp, sel.cpu().numpy()[:, :, :keff], None if out is None else out.cpu().numpy()


def check(cfg, inp, sel, out, bridge=0, heads=None, sorted_sets=False):
    heads = heads or [(b, hq) for b in range(cfg.B) for hq in range(cfg.Hq)]
    for b, hq in heads:
        r = head_oracle(inp, cfg, b, hq, cfg.N, bridge)
        got = np.sort(sel[b, hq]) if sorted_sets else sel[b, hq]
        np.testing.assert_array_equal(got, r["sel"], err_msg=f"top-K of query head {(b, hq)}")
        if out is not None:
            e = rel_l2(out[b, hq], r["out"][0])
            assert e <= OUT_RTOL, f"output row {(b, hq)} rel L2 {e}"


@pytest.mark.parametrize("G", [2, 4, 8])
def test_per_head_step_one_chunk(G):
    cfg = Config("ph", B=2, Hq=2 * G, Hkv=2, d=128, N=3000, L=300, K=200, bridge=0)
    inp, sel, out = run(cfg, 90 + G)
    check(cfg, inp, sel, out)


def test_per_head_heads_differ():
    """Per-head sets are not the GQA set: with G = 4 the four heads of a group select differently."""
    cfg = Config("ph", B=1, Hq=4, Hkv=1, d=128, N=3000, L=300, K=200, bridge=0)
    inp, sel, out = run(cfg, 95)
    assert any(not np.array_equal(sel[0, 0], sel[0, g]) for g in range(1, 4))
    check(cfg, inp, sel, out)


def test_per_head_select_only_long_context():
    cfg = Config("phl", B=2, Hq=8, Hkv=2, d=128, N=70000, L=512, K=int(np.ceil(0.06 * 70000)), bridge=0)
    inp, sel, out = run(cfg, 96, select_only=True)
    check(cfg, inp, sel, None, heads=[(0, 0), (0, 3), (1, 5), (1, 7)])


@pytest.mark.parametrize("frac", [0.9, 0.5])
def test_per_head_postings(frac):
    cfg = Config("php", B=2, Hq=8, Hkv=2, d=128, N=12000, L=300, K=800, bridge=0)
    inp, sel, out = run(cfg, 97, postings=frac, code_dist="zipf")
    check(cfg, inp, sel, out, sorted_sets=True)
    inp, sel, _ = run(cfg, 97, postings=frac, code_dist="zipf", select_only=True)
    check(cfg, inp, sel, None, sorted_sets=True)


def test_per_head_append_step():
    """Fused append (a0 + hist once) with G sub-steps == the per-head oracle on the final codes."""
    cfg = Config("pha", B=2, Hq=8, Hkv=2, d=128, N=5000, L=256, K=300, bridge=0)
    steps = 3
    inp = make_inputs(cfg, 98, device="cuda", family="g1", with_h=True, n_max=cfg.n_max(extra=steps + 8))
    params = A.Params(window=cfg.window, bridge=0, n_sink=cfg.n_sink, topk=cfg.K, group_reduce=PH)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], params)
    n0 = cfg.N - steps
    dec.encode(inp["k_cache"], 0, n0)
    sel = torch.full((cfg.B, cfg.Hq, cfg.K), -1, dtype=torch.int32, device="cuda")
    for s in range(steps):
        n = n0 + s + 1
        out = dec.step_append(inp["q"], inp["k_cache"], inp["v_cache"], n, sel_out=sel)
    torch.cuda.synchronize()
    # g1 keys are codewords: their codes are the drawn z (the oracle's input, not the GPU's codes)
    assert torch.equal(dec.codes[:, :, :cfg.N], inp["z"][:, :, :cfg.N].to(torch.uint16))
    codes = inp["z"][:, :, :cfg.N].to(torch.int64)
    h = torch.zeros_like(dec.hist).scatter_add_(2, codes, torch.ones_like(codes, dtype=torch.int32))
    assert torch.equal(h, dec.hist)               # a0 + histogram once per step, not once per head
    cpu = {k: (v.cpu() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    cpu["codes"] = inp["z"].cpu()
    check(cfg, cpu, sel.cpu().numpy(), out.cpu().numpy(), heads=[(0, 1), (1, 6), (1, 7)])


def test_per_head_repeated_steps_stable():
    """Stress for the sub-step plumbing: the gathered q of head position g is written by the kernel
    right before the sub-step, whose kernels read q before their dependency wait -- a gather that
    let its dependents launch early raced with them (seen as one head's stale selection)."""
    cfg = Config("phs", B=2, Hq=8, Hkv=2, d=128, N=12000, L=300, K=800, bridge=0)
    ref = None
    for rep in range(6):
        inp, sel, out = run(cfg, 97, postings=0.5, code_dist="zipf")
        if ref is None:
            ref = (sel, out)
            check(cfg, inp, sel, out, sorted_sets=True, heads=[(0, 2), (1, 2), (1, 7)])
        else:
            np.testing.assert_array_equal(sel, ref[0])
            assert np.array_equal(out.view(np.uint32), ref[1].view(np.uint32))


def test_per_head_with_uint8_codes_and_deferred_a0():
    """The variants compose: per-query-head selection over uint8 codes with the posting-list engine
    and a0 deferred (the newest 20 tokens not encoded) == the per-head oracle."""
    cfg = Config("phc", B=2, Hq=8, Hkv=2, d=128, N=6000, L=256, K=400, bridge=0)
    lag = 20
    inp = make_inputs(cfg, 99, device="cpu", family="g1", with_h=False)
    inp["codes"] = inp["z"].to(torch.uint16)
    dev = {k: (v.cuda() if isinstance(v, torch.Tensor) else v) for k, v in inp.items()}
    params = A.Params(window=cfg.window, bridge=0, n_sink=cfg.n_sink, topk=cfg.K, group_reduce=PH, hist_lag=lag)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], dev["codebook"], None, params, code_bytes=1)
    codes8 = dev["codes"].to(torch.int32).to(torch.uint8)
    codes8[:, :, cfg.N - lag:cfg.N] = 255 - codes8[:, :, cfg.N - lag:cfg.N]  # not encoded yet: garbage
    dec.codes = codes8
    c = dev["codes"][:, :, :cfg.N - lag].to(torch.int64)
    dec.hist = torch.zeros((cfg.B, cfg.Hkv, cfg.L), dtype=torch.int32, device="cuda")
    dec.hist.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
    dec.build_postings(cfg.N - cfg.window - 300)
    sel = torch.full((cfg.B, cfg.Hq, cfg.K), -1, dtype=torch.int32, device="cuda")
    out = dec.step_postings(dev["q"], dev["k_cache"], dev["v_cache"], cfg.N, sel_out=sel)
    torch.cuda.synchronize()
    check(cfg, inp, sel.cpu().numpy(), out.cpu().numpy(), sorted_sets=True, heads=[(0, 0), (0, 5), (1, 3), (1, 6)])
