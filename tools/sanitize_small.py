"""Small decode steps for compute-sanitizer runs (memcheck / racecheck / synccheck): the fused
one-chunk select, the long-context threshold + persistent scan, the split attention, the encode
roles and the sharded halves, at shapes that keep the instrumented run short.

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


run(Config("s1", B=1, Hq=4, Hkv=1, d=128, N=3000, L=256, K=100), 1)
run(Config("s2", B=2, Hq=8, Hkv=2, d=128, N=70001, L=512, K=4000), 2, long=True)
print("sanitize run ok")
