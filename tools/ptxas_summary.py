#!/usr/bin/env python
"""Summarise an nvcc -Xptxas -v log: kernel, registers, stack, spills, smem."""
import re
import subprocess
import sys

cur = None
rows = []
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["stack"], cur["spill_st"], cur["spill_ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
    m = re.search(r"(\d+) bytes smem", line)
    if m:
        cur["smem"] = int(m.group(1))
names = [r["name"] for r in rows]
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for r, d in zip(rows, dem):
    d = re.sub(r"lffn_gpu::", "", d)
    d = re.sub(r"\(.*\)$", "", d)
    print(f"{r.get('regs', '?'):>4} regs  stack {r.get('stack', 0):>4}  spill {r.get('spill_st', 0)}/{r.get('spill_ld', 0)}  smem {r.get('smem', 0):>6}  {d}")
