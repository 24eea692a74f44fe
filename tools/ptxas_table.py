"""Registers and spills per kernel from a `nvcc -Xptxas -v` log.

    python tools/ptxas_table.py build_ptxas.log [regex]
"""
import re
import sys

fn, pat = sys.argv[1], re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
cur, spill = None, ""
for line in open(fn):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = f"spill st {m.group(1):>4} ld {m.group(2):>4}"
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and pat.search(cur):
        print(f"{m.group(1):>4} regs  {spill}  {cur}")
        cur = None
