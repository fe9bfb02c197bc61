"""Timing of the offline codebook construction (a2ats_qavq_train) at the
paper's scale per KV head: L = 4096 codewords, d = 128, n keys and m post-PE queries
of a representative sample.  Prints one JSON line (seconds per head, per-phase estimates).

    python tools/train_bench.py [--n 65536] [--m 65536] [--L 4096] [--iters 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2502_12665_b200 import binding as Bd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--m", type=int, default=65536)
ap.add_argument("--L", type=int, default=4096)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
K = torch.randn((a.n, a.d), generator=g, device="cuda").to(torch.bfloat16)
Q = torch.randn((a.m, a.d), generator=g, device="cuda").to(torch.bfloat16)
u = torch.rand((a.L,), generator=g, device="cuda", dtype=torch.float64)
ws = torch.empty(Bd.a2ats_qavq_train_workspace_bytes(a.n, a.d, a.L, a.m), dtype=torch.uint8, device="cuda")
info = torch.zeros(2, dtype=torch.int32, device="cuda")
Bd.a2ats_qavq_train(K[:4096], 64, u[:64], 2, queries=Q[:4096], eps=1e-6)   # warm-up (attributes)
torch.cuda.synchronize()
res = {}
for name, iters in (("seed_only", 0), ("full", a.iters)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    Bd.a2ats_qavq_train(K, a.L, u, iters, queries=Q, eps=1e-6, info_out=info, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 1e3
it = int(info[0].item())
per_iter = (res["full"] - res["seed_only"]) / max(1, it)
flops_assign = 3.0 * a.n * a.L * a.d                   # (z - c)^2 accumulated per pair of (key, codeword)
print(json.dumps({"workload": "offline QAVQ codebook, one KV head", "n_keys": a.n, "m_queries": a.m, "L": a.L,
                  "d": a.d, "max_iters": a.iters, "iters_run": it, "seconds_per_head": res["full"],
                  "seconds_h_chol_z_kmeanspp": res["seed_only"], "seconds_per_lloyd_iteration": per_iter,
                  "assign_fp64_TFLOPs": flops_assign / per_iter / 1e12 if per_iter > 0 else None,
                  "dtype": "f64"}))
