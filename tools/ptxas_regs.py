"""Registers and spills per kernel from a ptxas -v log.  usage: python tools/ptxas_regs.py LOG [FILTER]"""
import re
import subprocess
import sys

cur = None
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill {m.group(1)}/{m.group(2)}"
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if flt in cur:
            print(f"{m.group(1):>4} regs  {spill:16s} {cur[:150]}")
        cur = None
