"""Which host<->device copy of bench.py's e2e loop costs what (C4 by default)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2502_12665_b200 as A  # noqa: E402
from synth import CONFIGS, budget_k, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
args = ap.parse_args()
cfg = CONFIGS[args.config]
inp = make_inputs(cfg, 3, device="cuda", with_h=True, n_max=cfg.n_max(extra=64))
q, kc, vc = inp["q"], inp["k_cache"], inp["v_cache"]
dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], A.Params(topk=budget_k(cfg.N)))
n0 = cfg.N - 20
dec.encode(kc, 0, n0)
B, Hq, Hkv, d = cfg.B, cfg.Hq, cfg.Hkv, cfg.d
q_host = q.cpu().pin_memory()
k_host = kc[:, :, n0].cpu().pin_memory()
v_host = vc[:, :, n0].cpu().pin_memory()
out_host = torch.empty((B, Hq, d), dtype=torch.float32).pin_memory()
q_dev = torch.empty_like(q)
k_stage = torch.empty((B, Hkv, d), dtype=torch.bfloat16, device="cuda")
out = torch.empty((B, Hq, d), dtype=torch.float32, device="cuda")


def variant(name, qc, kvc, oc, staged=False):
    def one(n):
        if qc:
            q_dev.copy_(q_host, non_blocking=True)
        if kvc:
            if staged:
                k_stage.copy_(k_host, non_blocking=True)
                kc[:, :, n - 1].copy_(k_stage)
                k_stage.copy_(v_host, non_blocking=True)
                vc[:, :, n - 1].copy_(k_stage)
            else:
                kc[:, :, n - 1].copy_(k_host, non_blocking=True)
                vc[:, :, n - 1].copy_(v_host, non_blocking=True)
        dec.params.topk = budget_k(n)
        dec.step_append(q_dev if qc else q, kc, vc, n, out=out)
        if oc:
            out_host.copy_(out, non_blocking=True)
    n = n0 + 1
    one(n)
    torch.cuda.synchronize()
    gs = []
    for s in range(6):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            one(n + 1 + s)
        gs.append(g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for g in gs:
        g.replay()
    e1.record()
    e1.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1) / len(gs) * 1e3:8.1f} us/step", flush=True)


variant("step only", False, False, False)
variant("+ q H2D", True, False, False)
variant("+ K/V rows H2D (strided)", False, True, False)
variant("+ K/V rows H2D (staged)", False, True, False, staged=True)
variant("+ out D2H", False, False, True)
variant("all (bench e2e)", True, True, True)
variant("all, staged K/V", True, True, True, staged=True)
