#!/usr/bin/env python3
"""Registers and spills per kernel from the build's ptxas -v logs.
    python tools/ptxas_regs.py [substring]"""
import glob
import os
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                    "paper_1611_02274_b200", "lib", "obj")
for f in sorted(glob.glob(os.path.join(root, "*.ptxas.txt"))):
    cur, spill = None, ""
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            spill = ""
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            spill = f"spill {m.group(1)}/{m.group(2)}" if m.group(1) != "0" else ""
        m = re.search(r"Used (\d+) registers", line)
        if m and cur and pat in cur:
            print(f"{m.group(1):>4} {spill:<16} {cur[:120]}")
