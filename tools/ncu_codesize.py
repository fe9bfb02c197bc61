import csv, sys, subprocess, io, re, collections
rep, kre, obj, mre = sys.argv[1:5]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Address" in r][0]
h = rows[hi]; ai = h.index("Address"); ie = h.index("Instructions Executed")
ex = []
for r in rows[hi + 1:]:
    if len(r) <= ie or not r[ai].startswith("0x"):
        if ex: break
        continue
    ex.append((int(r[ai], 16), float(r[ie] or 0)))
base = ex[0][0]
# line map via nvdisasm
import tempfile, glob, os
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = glob.glob(d + "/*.cubin")[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
fn = None; line = None; m = {}; want = None
for l in dis.splitlines():
    mm = re.search(r"\.text\.(\S+):", l)
    if mm: fn = mm.group(1); continue
    mm = re.search(r"line (\d+)", l)
    if "//##" in l and mm:
        fm = re.search(r'File "([^"]+)"', l)
        line = (os.path.basename(fm.group(1)) if fm else "?", int(mm.group(1))); continue
    mm = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if mm and fn and re.search(mre, fn):
        if want is None: want = fn
        if fn == want: m[int(mm.group(1), 16)] = line
cnt = collections.Counter(); dyn = collections.Counter()
for a, n in ex:
    off = a - base
    ln = m.get(off, ("?", 0))
    if n > 0: cnt[ln] += 1; dyn[ln] += n
tot = sum(cnt.values())
print("executed static instr", tot)
for k, v in cnt.most_common(40): print(f"{v:6d} {dyn[k]:12.0f} {k}")
