"""Small decode steps for compute-sanitizer runs (memcheck / racecheck / synccheck): the fused
one-chunk select, the long-context threshold + persistent scan, the split attention, the encode
roles, the posting-list select (list path with a short and a long unindexed tail, bitmap path,
fused append), the persistent LUT (B*G > 64), per-query-head sub-steps, uint8 codes and deferred
a0, at shapes that keep the instrumented run short.

    compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2502_12665_b200 as A  # noqa: E402
from synth import Config, make_inputs  # noqa: E402


def run(cfg, seed, long=False):
    inp = make_inputs(cfg, seed, device="cuda", with_h=True)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], A.Params(topk=cfg.K))
    dec.encode(inp["k_cache"], 0, cfg.N - 1)
    sel = torch.empty((cfg.B, cfg.Hkv, cfg.K), dtype=torch.int32, device="cuda")
    dec.step_append(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, sel_out=sel)
    dec.select(inp["q"], cfg.N, sel)
    dec.build_postings(cfg.N - 2)
    dec.select_postings(inp["q"], cfg.N, sel)
    torch.cuda.synchronize()


def run_postings(cfg, seed, group_reduce=0, code_bytes=2):
    inp = make_inputs(cfg, seed, device="cuda", with_h=True)
    dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"],
                    A.Params(topk=cfg.K, group_reduce=group_reduce), code_bytes=code_bytes)
    dec.encode(inp["k_cache"], 0, cfg.N - 1)
    G = 1 if group_reduce != 2 else cfg.Hq // cfg.Hkv
    sel = torch.empty((cfg.B, cfg.Hkv * G, cfg.K), dtype=torch.int32, device="cuda")
    for lag in (300, 3000, -1):  # short tail (staged path), long tail, index into the window (bitmap)
        dec.build_postings(cfg.N - 64 - lag if lag >= 0 else cfg.N - 2)
        dec.select_postings(inp["q"], cfg.N - 1, sel)
    dec.build_postings(cfg.N - 64 - 300)
    dec.step_append_postings(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, sel_out=sel)
    dec.params.hist_lag = 1
    dec.step_postings(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N + 1 if cfg.N + 1 <= inp["n_max"] else cfg.N,
                      sel_out=sel)
    torch.cuda.synchronize()


run(Config("s1", B=1, Hq=4, Hkv=1, d=128, N=3000, L=256, K=100), 1)
run(Config("s2", B=2, Hq=8, Hkv=2, d=128, N=70001, L=512, K=4000), 2, long=True)
run_postings(Config("p1", B=20, Hq=32, Hkv=8, d=128, N=9000, L=1024, K=540), 3)            # persistent LUT
run_postings(Config("p2", B=2, Hq=8, Hkv=2, d=128, N=9000, L=256, K=540), 4, group_reduce=2)  # per head
run_postings(Config("p3", B=2, Hq=8, Hkv=2, d=128, N=9000, L=256, K=540), 5, code_bytes=1)    # uint8 codes
print("sanitize run ok")
