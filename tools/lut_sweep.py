"""BASELINE configs[4]: codebook-size / top-K sweep of the score + top-K
path (a2ats_select_topk = a1..a4) at 32K-128K context, LUT on tensor cores vs FP32 FMA.

    python tools/lut_sweep.py [--out gpurun_out/lut_sweep.json] [--quick]

Per point: median device time of a CUDA-graph replay (L2 flushed before each replay,
outside the events) for lut_engine TENSOR and FMA, the approximate-scored tokens/s and the
score + top-K algorithmic bytes (codes once + codebook + Sel) against the measured HBM peak.
Synthetic inputs (synth/), codes uniform, hist maintained.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2502_12665_b200 as A  # noqa: E402
from synth.generators import _gen, make_codebook, make_codes, make_query  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "lut_sweep.json"))
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--quick", action="store_true")
args = ap.parse_args()

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
hbm = None
for k, v in peaks.items():
    if "hbm" in k.lower() and isinstance(v, (int, float)):
        hbm = float(v)
        break
hbm = hbm or 6545.3
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def time_point(B, N, L, K, engine, Hq=32, Hkv=8):
    g = _gen(7 + B + L + N, "cuda")
    n_max = (N + 63) // 64 * 64
    C = make_codebook(Hkv, L, 128, "g2", g, "cuda")
    q = make_query(B, Hq, 128, "g2", g, "cuda")
    codes = make_codes(B, Hkv, n_max, L, "uniform", g, "cuda").to(torch.uint16)
    c = codes[:, :, :N].to(torch.int64)
    hist = torch.zeros((B, Hkv, L), dtype=torch.int32, device="cuda")
    hist.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
    del c
    params = A.Params(topk=K, lut_engine=engine)
    shape = A.make_shape(B, Hq, Hkv, 128, L, n_max)
    ws = torch.zeros(A.a2ats_decode_workspace_bytes(shape, params), dtype=torch.uint8, device="cuda")
    keff = min(K, N - 68)
    sel = torch.empty((B, Hkv, max(keff, 1)), dtype=torch.int32, device="cuda")
    run = lambda: A.a2ats_select_topk(shape, params, N, q, codes, C, hist, sel, ws)  # noqa: E731
    run()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        run()
    ts = []
    for i in range(args.iters):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = statistics.median(ts)
    bytes_ = B * Hkv * N * 2 + Hkv * L * 128 * 2 + B * Hkv * keff * 4
    return {"us": us, "tokens_per_s": B * Hkv * N / (us * 1e-6), "hbm_frac": bytes_ / (us * 1e-6) / 1e9 / hbm,
            "lut_flops": 2 * B * Hq * L * 128}


res = {"hbm_peak_GBps": hbm, "points": []}
Bs = [1, 16, 64] if args.quick else [1, 4, 16, 64]
Ls = [256, 1024, 4096]
Ns = [32768, 131072]
for N in Ns:
    for L in Ls:
        for B in Bs:
            if B * N > 64 * 131072:
                continue
            K = -(-6 * N // 100)
            row = {"B": B, "N": N, "L": L, "K": K, "BGL": B * 4 * L}
            for eng, name in ((1, "tensor"), (2, "fma")):
                row[name] = time_point(B, N, L, K, eng)
            row["faster"] = "tensor" if row["tensor"]["us"] < row["fma"]["us"] else "fma"
            res["points"].append(row)
            print(json.dumps({k: (v if not isinstance(v, dict) else round(v["us"], 1)) for k, v in row.items()}),
                  flush=True)
# top-K sweep at Llama-3.1-8B 128K shapes (B = 64, L = 4096): K = 1..10 % of N
for pct in ([1, 6, 10] if args.quick else [1, 2, 3, 6, 10]):
    N, L, B = 131072, 4096, 64
    K = -(-pct * N // 100)
    r = time_point(B, N, L, K, 0)
    res["points"].append({"B": B, "N": N, "L": L, "K": K, "K_pct": pct, "auto": r})
    print(json.dumps({"K_pct": pct, "us": round(r["us"], 1), "hbm_frac": round(r["hbm_frac"], 3)}), flush=True)
os.makedirs(os.path.dirname(args.out), exist_ok=True)
json.dump(res, open(args.out, "w"), indent=1)
print("wrote", args.out)
