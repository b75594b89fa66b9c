"""Opcode histogram of the main row loop (largest BRA.U back edge) of one kernel's SASS.
usage: python tools/loop_hist.py LIB.so MANGLED_NAME_SUBSTRING"""
import collections
import re
import subprocess
import sys

lib, name = sys.argv[1], sys.argv[2]
FULL = len(sys.argv) > 3
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
body, on = [], False
for l in sass.splitlines():
    if "Function :" in l:
        on = name in l
        continue
    if on:
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
        if m:
            body.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for a, ins in body:
    m = re.search(r'BRA\.U\s+!?UP\d,\s*0x([0-9a-f]+)', ins)
    if m and int(m.group(1), 16) < a:
        t = int(m.group(1), 16)
        if best is None or a - t > best[1] - best[0]:
            best = (t, a)
ops = collections.Counter()
for a, ins in body:
    if best[0] <= a <= best[1]:
        if ins.startswith('@'):
            ins = ins.split(None, 1)[1]
        op = ins.split()[0]
        ops[op if (FULL or op.startswith(("LDS", "STS"))) else op.split(".")[0]] += 1
print(hex(best[0]), hex(best[1]), "total", sum(ops.values()))
print(" ".join(f"{k}:{v}" for k, v in ops.most_common(40)))
