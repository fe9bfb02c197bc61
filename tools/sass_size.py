"""Instruction count per kernel in a built library (code-size / I-cache check).

    python tools/sass_size.py [paper_2502_12665_b200/lib/liba2ats.so]
"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2502_12665_b200/lib/liba2ats.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, counts = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = 0
        continue
    if cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", line):
        counts[cur] += 1
for k, v in sorted(counts.items(), key=lambda kv: -kv[1]):
    name = re.sub(r"_GLOBAL__N__\w+?_\d+_(\w+?)_cu_\w+?\d+", r"\1:", k)
    print(f"{v:6d} instr {v * 16 / 1024:7.1f} KB  {name[:110]}")
