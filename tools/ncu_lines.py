"""Per-source-line warp-stall samples of one kernel in an ncu report (SASS page
mapped to CUDA lines through nvdisasm -g of the same object).

    python tools/ncu_lines.py REP KERNEL_REGEX OBJ MANGLED_REGEX [top]
"""
import csv
import io
import re
import subprocess
import sys
import glob
import os
import tempfile

rep, kre, obj = sys.argv[1], sys.argv[2], sys.argv[3]
mre = sys.argv[4]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Address" in r][0]
h = rows[hi]
ai, si, ns = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed") if "Instructions Executed" in h else None
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
wf_i = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
wfi_i = h.index("L1 Wavefronts Shared Ideal") if "L1 Wavefronts Shared Ideal" in h else None
kname = rows[0][1] if len(rows[0]) > 1 else ""
samples = []
for r in rows[hi + 1:]:
    if len(r) <= ns or not r[ai].startswith("0x"):
        if samples:
            break  # first kernel instance only
        continue
    st = {c: int(float(r[i] or 0)) for i, c in stall_cols}
    wf = (float(r[wf_i] or 0), float(r[wfi_i] or 0)) if wf_i is not None else (0.0, 0.0)
    st["_inst"] = int(float(r[ie] or 0)) if ie is not None else 0
    samples.append((int(r[ai], 16), r[si], int(float(r[ns] or 0)), st, wf))
base = samples[0][0]
# offset -> line from nvdisasm of the matching function
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
fn_pat = re.compile(r"\.text\.(\S+):")
cur, line, lmap = None, None, {}
fname = None
want = None
for l in dis.splitlines():
    m = fn_pat.search(l)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"line (\d+)", l)
    if "//##" in l and m:
        fm = re.search(r'File "([^"]+)"', l)
        line = (os.path.basename(fm.group(1)) if fm else "?", int(m.group(1)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and cur and re.search(mre, cur):
        if want is None:
            want = cur
        if cur == want:
            lmap[int(m.group(1), 16)] = line
agg = {}
tot = 0
for addr, src, n, st, wf in samples:
    ln = lmap.get(addr - base)
    e = agg.setdefault(ln, [0, src, {}, [0.0, 0.0]])
    e[0] += n
    for c, v in st.items():
        e[2][c] = e[2].get(c, 0) + v
    e[3][0] += wf[0]
    e[3][1] += wf[1]
    tot += n
tot_inst = sum(st["_inst"] for _, _, _, st, _ in samples)
print(f"kernel {kname}  function {want}  total samples {tot}  warp instructions {tot_inst}")
src_lines = None
srcfile = None
srcpath = None
for l in dis.splitlines():
    m = re.search(r'File "([^"]+)"', l)
    if m and os.path.exists(m.group(1)):
        srcpath = m.group(1)
        break
lines = open(srcpath).read().splitlines() if srcpath else []
for ln, (n, s, st, wf) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    f, n_ = ln if ln else ("?", 0)
    txt = lines[n_ - 1].strip()[:80] if srcpath and f == os.path.basename(srcpath) and 0 < n_ <= len(lines) else f
    inst = st.pop("_inst", 0)
    top2 = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    why = " ".join(f"{c[6:]}:{v}" for c, v in top2 if v)
    smem = f" smem-wf {wf[0]:.0f}/{wf[1]:.0f}" if wf[0] else ""
    print(f"{n:6d} {100.0 * n / max(tot, 1):5.1f}% inst {100.0 * inst / max(tot_inst, 1):5.1f}%  {n_}: {txt}  [{why}]{smem}")
