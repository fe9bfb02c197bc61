"""Kernel micro-benchmark for ncu / quick timing: C2-shaped decode steps through the C ABI.

    python tools/kbench.py [--config C2] [--iters 5] [--no-hist] [--encode]
Not the bench contract (see bench.py); used for ncu captures and per-kernel timing.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2502_12665_b200 as A  # noqa: E402
from synth import CONFIGS, budget_k, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--no-hist", action="store_true")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--L", type=int, default=0)
ap.add_argument("--N", type=int, default=0)
ap.add_argument("--select-only", action="store_true", help="a2ats_select_topk (a1..a4) only")
ap.add_argument("--postings", action="store_true", help="posting-list selection engine (f3)")
ap.add_argument("--post-lag", type=int, default=256, help="tokens behind the window start the index was built at")
ap.add_argument("--no-append", action="store_true", help="step without a0 (codes / hist given for all tokens)")
ap.add_argument("--encode-batch", type=int, default=0, help="also time a2ats_build_codes of this many tokens per pair")
args = ap.parse_args()
cfg = CONFIGS[args.config]
if args.batch:
    cfg = cfg.with_(B=args.batch)
if args.L:
    cfg = cfg.with_(L=args.L)
if args.N:
    cfg = cfg.with_(N=args.N, K=budget_k(args.N))
inp = make_inputs(cfg, 5, device="cuda", with_h=True)
codes = inp["z"].to(torch.uint16)
hist = torch.zeros((cfg.B, cfg.Hkv, cfg.L), dtype=torch.int32, device="cuda")
c = codes[:, :, :cfg.N].to(torch.int64)
hist.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], A.Params(topk=cfg.K))
dec.codes, dec.hist = codes, hist
out = torch.empty((cfg.B, cfg.Hq, 128), device="cuda")
scratch_codes = torch.zeros_like(codes)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
for e in evs:
    e.record()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
hist0 = hist.clone()
c0 = codes[:, :, :cfg.N - 1].to(torch.int64)
hist0.zero_().scatter_add_(2, c0, torch.ones_like(c0, dtype=torch.int32))
sel_buf = torch.empty((cfg.B, cfg.Hkv, max(cfg.K, 1)), dtype=torch.int32, device="cuda")
if args.postings:
    for it in range(3):
        flush.fill_(it)
        e0.record()
        dec.build_postings(cfg.N - cfg.window - args.post_lag)
        e1.record()
        torch.cuda.synchronize()
        print("postings_build %.1f us" % (e0.elapsed_time(e1) * 1e3))
for it in range(args.iters if args.select_only else 0):
    flush.fill_(it)
    e0.record()
    if args.postings:
        dec.select_postings(inp["q"], cfg.N, sel_buf)
    else:
        dec.select(inp["q"], cfg.N, sel_buf)
    e1.record()
    torch.cuda.synchronize()
    print("it", it, "select_topk %.1f us" % (e0.elapsed_time(e1) * 1e3))
for it in range(0 if args.select_only else args.iters):
    flush.fill_(it)
    dec.hist.copy_(hist0)  # covers [0, N-1): the step appends token N-1
    e0.record()
    A.a2ats_set_stage_events(evs)
    if args.postings and args.no_append:
        dec.hist.copy_(hist)
        dec.step_postings(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, out=out)
    elif args.postings:
        dec.step_append_postings(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, out=out)
    elif args.no_append:
        dec.hist.copy_(hist)
        dec.step(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, out=out, use_hist=not args.no_hist)
    else:
        dec.step_append(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, out=out, use_hist=not args.no_hist)
    A.a2ats_set_stage_events(None)
    e1.record()
    torch.cuda.synchronize()
    names = ["prep", "select", "attn", "tail"]
    print("it", it, "step %.1f" % (e0.elapsed_time(e1) * 1e3), " ".join(
        "%s %.1f" % (n, evs[i].elapsed_time(evs[i + 1]) * 1e3) for i, n in enumerate(names)), "us")

if args.encode_batch:
    T = args.encode_batch
    for it in range(4):
        flush.fill_(it)
        e0.record()
        dec.encode(inp["k_cache"], cfg.N - T, cfg.N, update_hist=True, codes=scratch_codes)
        e1.record()
        torch.cuda.synchronize()
        print("build_codes %d tokens/pair %.1f us" % (T, e0.elapsed_time(e1) * 1e3))
