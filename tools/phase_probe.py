"""Phase timing of CTA 0 of the select kernel (tuning build liba2ats_phases.so, A2ATS_PHASES)."""
import ctypes
import os
import sys

os.environ.setdefault("A2ATS_LIB", os.path.join(os.path.dirname(__file__), "..", "paper_2502_12665_b200", "lib",
                                                "liba2ats_phases.so"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import paper_2502_12665_b200 as A  # noqa: E402
from synth import CONFIGS, make_inputs  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
inp = make_inputs(cfg, 5, device="cuda", with_h=False)
codes = inp["z"].to(torch.uint16)
hist = torch.zeros((cfg.B, cfg.Hkv, cfg.L), dtype=torch.int32, device="cuda")
c = codes[:, :, :cfg.N].to(torch.int64)
hist.scatter_add_(2, c, torch.ones_like(c, dtype=torch.int32))
dec = A.Decoder(cfg.B, cfg.Hq, cfg.Hkv, cfg.L, inp["n_max"], inp["codebook"], None, A.Params(topk=cfg.K))
dec.codes, dec.hist = codes, hist
lib = A.load()
lib.a2ats_debug_select_phases.argtypes = [ctypes.POINTER(ctypes.c_longlong)]
buf = (ctypes.c_longlong * 16)()
for it in range(3):
    dec.step(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N)
    torch.cuda.synchronize()
    lib.a2ats_debug_select_phases(buf)
    t0 = buf[0]
    print("it", it, " ".join(f"p{i}:{(buf[i]-t0)/1.9e3:.2f}us" for i in range(12) if buf[i]))

# LUT kernel phases (CTA 0), if exported by this build
if hasattr(lib, "a2ats_debug_lut_phases"):
    lib.a2ats_debug_lut_phases.argtypes = [ctypes.POINTER(ctypes.c_longlong)]
    for it in range(2):
        dec.step(inp["q"], inp["k_cache"], inp["v_cache"], cfg.N)
        torch.cuda.synchronize()
        lib.a2ats_debug_lut_phases(buf)
        t0 = buf[0]
        print("lut it", it, " ".join(f"p{i}:{(buf[i]-t0)/1.9e3:.2f}us" for i in range(8) if buf[i]))
