"""Per-CTA start/end timeline of each kernel of one encode + decode step
(tuning build liba2ats_phases.so: thread 0 of every CTA records %globaltimer).

    python tools/timeline_probe.py [--config C2] [--iters 3]
Prints, per kernel, relative to the first CTA start of the step: first/last CTA
start, first/last CTA end, and the CTA duration quantiles; for the attention, the
slowest CTAs as (split, pair).
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("A2ATS_LIB", os.path.join(ROOT, "paper_2502_12665_b200", "lib", "liba2ats_phases.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_12665_b200 as A  # noqa: E402
from synth import CONFIGS, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--select-only", action="store_true", help="a2ats_select_topk (a1..a4) instead of the step")
ap.add_argument("--postings", action="store_true", help="select-only through the posting-list engine (f3)")
ap.add_argument("--graph", action="store_true", help="the postings select replayed from a CUDA graph")
args = ap.parse_args()
cfg = CONFIGS[args.config]
inp = make_inputs(cfg, 5, device="cuda", with_h=True)
codes = inp["z"].to(torch.uint16)
hist = torch.zeros((cfg.B, cfg.Hkv, cfg.L), dtype=torch.int32, device="cuda")
c = codes[:, :, :cfg.N].to(torch.int64)
hist.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], inp["H"], A.Params(topk=cfg.K))
dec.codes, dec.hist = codes, hist
hist0 = torch.zeros_like(hist)
c0 = codes[:, :, :cfg.N - 1].to(torch.int64)
hist0.scatter_add_(2, c0, torch.ones_like(c0, dtype=torch.int32))
scratch = torch.zeros_like(codes)
out = torch.empty((cfg.B, cfg.Hq, 128), device="cuda")
lib = A.load()
KMAX = 8192
kernels = ["prep", "select", "selc"] if args.select_only else ["prep", "select", "selc", "attn"]
if args.postings:
    kernels = ["prep", "select", "selp"]
sel_buf = torch.empty((cfg.B, cfg.Hkv, cfg.K), dtype=torch.int32, device="cuda")
fns = {}
for k in kernels:
    f = getattr(lib, f"a2ats_debug_{k}_timeline")
    f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    fns[k] = f
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
if args.postings:
    args.select_only = True
    dec.build_postings(cfg.N - cfg.window - 256)
ncta = {}
g_post = None
if args.postings and args.graph:
    dec.select_postings(inp["q"], cfg.N, sel_buf)
    torch.cuda.synchronize()
    g_post = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_post):
        dec.select_postings(inp["q"], cfg.N, sel_buf)
    torch.cuda.synchronize()
for it in range(args.iters):
    flush.fill_(it)
    dec.hist.copy_(hist if args.select_only else hist0)  # step: covers [0, N-1), the step appends N-1
    if g_post is not None:
        g_post.replay()
    elif args.postings:
        dec.select_postings(inp["q"], cfg.N, sel_buf)
    elif args.select_only:
        dec.select(inp["q"], cfg.N, sel_buf)
    else:
        dec.step_append(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N, out=out)
    torch.cuda.synchronize()
    tl = {}
    for k in kernels:
        buf = (ctypes.c_ulonglong * (8 * KMAX))()
        fns[k](buf)
        arr = np.frombuffer(buf, dtype=np.uint64).reshape(KMAX, 8).astype(np.int64)
        tl[k] = arr
    if it == 0:
        continue
    # CTAs written in this step: end >= start and start after the previous marks
    valid = {}
    for k in kernels:
        a = tl[k]
        last = a[:, 0].max()
        m = (a[:, 0] > last - 2_000_000) & (a[:, 1] >= a[:, 0]) & (a[:, 0] > 0)  # this step's CTAs
        if k == "prep":
            m[4096:] = False  # (qprep rows)
        valid[k] = np.nonzero(m)[0]
    t0 = min(tl[k][valid[k], 0].min() for k in kernels if len(valid[k]))
    print(f"--- iter {it} (us from first CTA start)")
    for k in kernels:
        if not len(valid[k]):
            continue
        a = tl[k][valid[k]]
        st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
        du = en - st
        q = np.percentile(du, [0, 50, 90, 100])
        print(f"{k:7s} ctas {len(a):5d} start {st.min():7.2f}..{st.max():7.2f} end {en.min():7.2f}..{en.max():7.2f}"
              f"  dur min/med/p90/max {q[0]:6.2f} {q[1]:6.2f} {q[2]:6.2f} {q[3]:6.2f}")
    qp = tl["prep"][4096:4096 + 256]
    qp = qp[(qp[:, 0] > 0) & (qp[:, 1] >= qp[:, 0]) & (qp[:, 0] > tl["prep"][:, 0].max() - 2_000_000)]
    if len(qp):
        print(f"  qprep ctas {len(qp)} start {(qp[:, 0].min() - t0) / 1e3:.2f}..{(qp[:, 0].max() - t0) / 1e3:.2f}"
              f" wait-ret {(qp[:, 2].min() - t0) / 1e3:.2f}..{(qp[:, 2].max() - t0) / 1e3:.2f}"
              f" end {(qp[:, 1].min() - t0) / 1e3:.2f}..{(qp[:, 1].max() - t0) / 1e3:.2f}")
    if args.postings:  # persistent LUT marks: 2 wait, 3 first unit's accumulator, 4 first epilogue, 5 last accumulator, 6 last epilogue
        r = tl["prep"][valid["prep"]]
        d = lambda x, y: np.percentile((r[:, x] - r[:, y]) / 1e3, [10, 50, 90]).round(2)
        print("  lut_persist (p10/p50/p90): setup+wait", d(2, 0), " first A", d(6, 2), " first B", d(7, 2),
              " first mma", d(3, 7), " first epi", d(4, 3), " to last mma", d(5, 4), " last epi+end", d(1, 5))
    # prep roles (slot 7: 1 LUT, 2 encode, 3 window)
    pa, pidx = tl["prep"], valid["prep"]
    for name, role in (("lut", 1), ("encode", 2), ("window", 3)):
        sel = pidx[pa[pidx, 7] == role]
        if len(sel):
            st, en = (pa[sel, 0] - t0) / 1e3, (pa[sel, 1] - t0) / 1e3
            extra = ""
            if role == 3:
                r = pa[sel]
                d = lambda x, y: np.median((r[:, x] - r[:, y]) / 1e3)
                extra = (f"  [cs {d(2, 0):.2f}  1st pair loads {d(3, 2):.2f}  compute {d(4, 3):.2f}"
                         f"  wait {d(5, 4):.2f}  rest {d(1, 5):.2f}]")
            if role == 1:
                r = pa[sel]
                d = lambda x, y: np.median((r[:, x] - r[:, y]) / 1e3)
                extra = (f"  [q~ {d(2, 0):.2f}  wait {d(3, 2):.2f}  cs {d(4, 3):.2f}  mma1 {d(5, 4):.2f}"
                         f"  epi1 {d(6, 5):.2f}  rest {d(1, 6):.2f}]")
            print(f"  prep/{name:6s} ctas {len(sel):4d} start {st.min():7.2f}..{st.max():7.2f} end {en.min():7.2f}..{en.max():7.2f}"
                  f"  dur med {np.median(en - st):6.2f}{extra}")
    m = tl["select"][valid["select"]]
    m = m[(m[:, 3] > m[:, 0]) & (m[:, 2] > m[:, 3])]
    if len(m):  # stream kernel marks: 3 = dependency wait returned, 2 = class table built
        d = lambda x, y: np.median((m[:, x] - m[:, y]) / 1e3)
        print(f"  select phases (median us): start->wait {d(3, 0):.2f}  threshold+table {d(2, 3):.2f}"
              f" [keys {d(4, 3):.2f} level {d(5, 4):.2f} table {d(2, 5):.2f}]"
              f"  stream {d(1, 2):.2f}  (wait returns {(m[:, 3].min() - t0) / 1e3:.2f}..{(m[:, 3].max() - t0) / 1e3:.2f})")
    m = tl["select"][valid["select"]]
    if args.postings and len(m):  # postings kernel marks: 2 wait, 3 level, 6 bounds+scan, 7 table, 4 copy, 5 tail+ties
        d = lambda x, y: np.percentile((m[:, x] - m[:, y]) / 1e3, [10, 50, 90]).round(2)
        print("  postings (p10/p50/p90 us): start->wait", d(2, 0), " level", d(3, 2), " bounds+scan", d(6, 3),
              " table", d(7, 6), " copy", d(4, 7), " tail+ties", d(5, 4), " end", d(1, 5))
        print("    wait returns", np.percentile((m[:, 2] - t0) / 1e3, [0, 50, 100]).round(2))
        p2 = tl["selp"][valid["select"]]
        mm = np.concatenate([m, p2], axis=1)  # columns 8.. = selp marks
        d = lambda x, y: np.percentile((mm[:, x] - mm[:, y]) / 1e3, [10, 50, 90]).round(2)
        print("    prologue: loads", d(8, 0), " corrections", d(9, 8), " wait", d(2, 9))
        print("    level: range", d(5, 2), " bins+pick", d(6, 5), " survivors", d(7, 6), " rank", d(3, 7))
        print("    after: classes", d(10, 3), " sink-skip", d(11, 10), " q_scan", d(12, 11), " table", d(13, 12),
              " copy", d(14, 13), " tail+ties", d(15, 14), " end", d(1, 15))
    elif len(m) and (m[:, 4] > m[:, 3]).all():  # threshold kernel marks: 3 wait returned, 4 level found
        d = lambda x, y: np.percentile((m[:, x] - m[:, y]) / 1e3, [10, 50, 90]).round(2)
        print("  thresh (p10/p50/p90 us): start->wait", d(3, 0), " keys+level", d(4, 3), " table+E", d(1, 4))
        print("    keys", d(5, 3), " bins+pick", d(6, 5), " survivors", d(7, 6), " rank", d(4, 7))
    m = tl["selc"][valid["selc"]] if "selc" in valid and len(valid["selc"]) else []
    if len(m) and (m[:, 3] > m[:, 2]).all():  # scan kernel marks: 2 wait returned, 3 first unit done
        d = lambda x, y: np.percentile((m[:, x] - m[:, y]) / 1e3, [10, 50, 90]).round(2)
        print("  scan (p10/p50/p90 us): start->wait", d(2, 0), " unit0", d(3, 2), " rest", d(1, 3))
        print("    unit0: table0", d(4, 2), " sr1 classify+scan", d(5, 4), " barrier", d(6, 5), " sr1 emit", d(7, 6),
              " sr2 + unit end", d(3, 7))
    if args.select_only:
        continue
    if len(valid["selc"]):
        m = tl["selc"][valid["selc"]]
        m = m[(m[:, 4] > m[:, 0])]
        if len(m):
            d = lambda x, y: np.median((m[:, x] - m[:, y]) / 1e3)
            print(f"  selc phases (median us): wait+table {d(2, 0):.2f}  classify {d(3, 2):.2f}  lookback {d(4, 3):.2f}"
                  f"  emit+exit {d(1, 4):.2f}")
    a = tl["attn"]
    idx = valid["attn"]
    du = (a[idx, 1] - a[idx, 0]) / 1e3
    order = np.argsort(-du)[:8]
    # attention grid is (nsplit_max, P): linear id = pair * gridDim.x + split
    nsx = int(idx.max() + 1) // (cfg.B * cfg.Hkv)
    print("  slowest attn CTAs (split, pair, us):",
          [(int(idx[o] % nsx), int(idx[o] // nsx), round(float(du[o]), 2)) for o in order])
    print("  attn CTA duration by split:", {s: round(float(np.median(du[(idx % nsx) == s])), 2) for s in range(nsx)})
    # phase marks: 2 = index prologue done (after the dependency wait), 3 = main loop done,
    # 4 = last-arriver combine start (only the last CTA of a pair)
    for sp in range(nsx):
        rows = a[idx[(idx % nsx) == sp]]
        pro = np.median((rows[:, 2] - rows[:, 0]) / 1e3)
        loop = np.median((rows[:, 3] - rows[:, 2]) / 1e3)
        tail = np.median((rows[:, 1] - rows[:, 3]) / 1e3)
        last = rows[rows[:, 4] > rows[:, 0]]
        comb = np.median((last[:, 1] - last[:, 4]) / 1e3) if len(last) else float("nan")
        print(f"  split {sp}: start->prologue {pro:.2f}  loop {loop:.2f}  loop->end {tail:.2f}  "
              f"last-arrivers {len(last)} combine {comb:.2f} us")
