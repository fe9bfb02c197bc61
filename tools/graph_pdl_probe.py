"""Does a CUDA graph that contains PDL launches from liba2ats.so + event records time correctly?"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2502_12665_b200 as A
from synth import CONFIGS, make_inputs, budget_k

cfg = CONFIGS["C2"]
inp = make_inputs(cfg, 5, device="cuda", with_h=True, n_max=cfg.n_max(extra=64))
dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], A.Params(topk=budget_k(cfg.N + 64)))
dec.encode(inp["k_cache"], 0, cfg.N - 10)
out = torch.empty((cfg.B, cfg.Hq, 128), device="cuda")
n = cfg.N - 10
def step(n):
    dec.encode(inp["k_cache"], n - 1, n)
    dec.params.topk = budget_k(n)
    dec.step(inp["q"], inp["k_cache"], inp["v_cache"], n, out=out)
n += 1; step(n); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
# events inside the graph
g = torch.cuda.CUDAGraph()
n += 1
with torch.cuda.graph(g):
    e0.record(); step(n); e1.record()
torch.cuda.synchronize()
try:
    g.replay(); torch.cuda.synchronize()
    print("inside-graph events:", e0.elapsed_time(e1) * 1e3, "us")
except Exception as ex:
    print("inside-graph events FAILED:", repr(ex)[:200])
torch.cuda.synchronize()
# events outside the graph
g2 = torch.cuda.CUDAGraph()
n += 1
with torch.cuda.graph(g2):
    step(n)
f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(3):
    f0.record(); g2.replay(); f1.record(); torch.cuda.synchronize()
    print("outside-graph events:", f0.elapsed_time(f1) * 1e3, "us")
