import sys, os, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_2502_12665_b200 as A
from synth.generators import _gen, make_codebook, make_codes, make_query
flush = torch.empty(64*1024*1024, dtype=torch.float32, device="cuda")
for B in (1, 4, 8, 16):
  for eng in (1, 2):
    N, L, Hq, Hkv = 32768, 1024, 32, 8
    g = _gen(7, "cuda")
    n_max = N + 64
    C = make_codebook(Hkv, L, 128, "g2", g, "cuda"); q = make_query(B, Hq, 128, "g2", g, "cuda")
    codes = make_codes(B, Hkv, n_max, L, "uniform", g, "cuda").to(torch.uint16)
    c = codes[:, :, :N].to(torch.int64); hist = torch.zeros((B, Hkv, L), dtype=torch.int32, device="cuda"); hist.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
    params = A.Params(topk=1967, lut_engine=eng); shape = A.make_shape(B, Hq, Hkv, 128, L, n_max)
    ws = torch.zeros(A.a2ats_decode_workspace_bytes(shape, params), dtype=torch.uint8, device="cuda")
    sel = torch.empty((B, Hkv, 1967), dtype=torch.int32, device="cuda")
    run = lambda: A.a2ats_select_topk(shape, params, N, q, codes, C, hist, sel, ws)
    run(); torch.cuda.synchronize()
    ts = []
    for i in range(10):
        flush.fill_(i); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1e3)
    print(B, "tensor" if eng == 1 else "fma", round(statistics.median(ts), 1), flush=True)
