"""Registers / spills per kernel from csrc/ptxas.log (or a given log): python tools/ptxas_summary.py [LOG] [FILTER]"""
import re
import sys

log = sys.argv[1] if len(sys.argv) > 1 else "paper_1802_04243_b200/csrc/ptxas.log"
flt = sys.argv[2] if len(sys.argv) > 2 else ""
name = None
spill = ""
for l in open(log):
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", l)
    if m:
        spill = m.group(1)
    m = re.search(r"Used (\d+) registers", l)
    if m and name and flt in name:
        print(f"{m.group(1):>4} regs  spill {spill:>4}  {name}")
        name = None
