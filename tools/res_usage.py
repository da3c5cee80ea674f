"""Registers / stack per kernel of a built library: python tools/res_usage.py lib.so [regex]"""
import re
import subprocess
import sys

out = subprocess.check_output(["cuobjdump", "-res-usage", sys.argv[1]], text=True)
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
name = None
for line in out.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+)", line)
    if m and name:
        dn = subprocess.check_output(["c++filt", name], text=True).strip().split("(")[0]
        if pat is None or pat.search(dn):
            print(f"{dn:60s} REG {m.group(1):>3s} STACK {m.group(2):>4s} SHARED {m.group(3)}")
        name = None
