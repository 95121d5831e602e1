#!/usr/bin/env python
"""Registers / stack of the stream-collide kernels in liblbm.so's objects (cuobjdump
-res-usage), demangled:  python scripts/regs.py [object-glob] [kernel-substring]"""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pat = sys.argv[1] if len(sys.argv) > 1 else "ops_*.o"
sub = sys.argv[2] if len(sys.argv) > 2 else "k_"
for obj in sorted(glob.glob(os.path.join(ROOT, "paper_2211_02435_b200", "build", pat))):
    out = subprocess.run(["cuobjdump", "-res-usage", obj], capture_output=True, text=True).stdout
    names, regs = [], []
    fn = None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+)", line)
        if m and fn:
            names.append(fn)
            regs.append((int(m.group(1)), int(m.group(2))))
            fn = None
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    for d, (r, st) in zip(dem, regs):
        if sub in d:
            print(f"{r:4d} {st:4d}  {d.split('(')[0]}")
