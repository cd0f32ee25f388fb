"""Registers / spills per kernel from a ptxas -v log:
    python scripts/ptxas_spills.py paper_2603_28770_b200/csrc/build/bfgs_wide.o.ptxas.log [filter]"""
import re
import subprocess
import sys

cur = None
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '([^']+)'", line) or re.search(
        r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        name = subprocess.run(["c++filt"], input=cur, capture_output=True, text=True).stdout.strip()
        if flt in name:
            print(f"{m2.group(1):>4s} regs  spill st/ld {spill[0]:4d}/{spill[1]:4d}  {name[:110]}")
