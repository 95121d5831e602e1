#!/usr/bin/env python
"""Compiled fp64/fp32 arithmetic per cell update of every stream-collide kernel,
counted from the SASS of liblbm.so's objects (cuobjdump), the compiled analogue of
the paper's symbolic op counts (Table 1) and of the savings from
regularisation (Table 2).  Straight-line kernels: every counted
instruction executes once per cell (the instruction counts are per thread = per cell).

  python scripts/sass_opcount.py [--markdown]
"""
from __future__ import annotations

import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2211_02435_b200", "build")

FP64 = ("DFMA", "DADD", "DMUL")
FP32 = ("FFMA", "FADD", "FMUL")
SPACES = {0: "POP", 1: "RAW", 2: "CM", 3: "K", 4: "SWE-CM", 5: "SWE-K"}
REGS = {0: "abs", 1: "zc+delta", 2: "zc+eq"}
RSN = {0: "general", 1: "R- (all but shear = 1)", 2: "HO (orders 5,6 = 1)"}


def demangle(names):
    p = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return p.stdout.splitlines()


def count(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\d\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            op = m.group(1).split(".")[0]
            funcs[cur][op] += 1
    return funcs


def main():
    rows = []
    for obj in sorted(glob.glob(os.path.join(OBJ, "ops_*.o"))):
        funcs = count(obj)
        names = list(funcs)
        for mangled, dem in zip(names, demangle(names)):
            m = re.match(r"void lbm::k_pull<lbm::(D\dQ\d+), (\d), (\d), (double|float), false, (\d)>", dem)
            if not m:
                continue
            st, sp, reg, real, rs = m.group(1), int(m.group(2)), int(m.group(3)), m.group(4), int(m.group(5))
            c = funcs[mangled]
            ops = FP64 if real == "double" else FP32
            n = {k: c[k] for k in ops}
            total = sum(n.values())
            flops = sum(2 * c[k] if k.endswith("FMA") else c[k] for k in ops)
            rows.append((st, SPACES[sp], REGS[reg], real, RSN[rs], n, total, flops, c["LDG"], c["STG"]))
    rows.sort()
    md = "--markdown" in sys.argv
    if md:
        print("| stencil | space | regime | real | rates | FMA | ADD | MUL | fp instr/cell | flop/cell |")
        print("|---|---|---|---|---|---|---|---|---|---|")
    for st, sp, reg, real, rs, n, total, flops, ldg, stg in rows:
        k = list(n.values())
        if md:
            print(f"| {st} | {sp} | {reg} | {real} | {rs} | {k[0]} | {k[1]} | {k[2]} | {total} | {flops} |")
        else:
            print(f"{st:6s} {sp:4s} {reg:9s} {real:6s} {rs:24s} fma {k[0]:4d} add {k[1]:4d} mul {k[2]:4d} "
                  f"instr {total:4d} flop {flops:5d}  ldg {ldg} stg {stg}")


if __name__ == "__main__":
    main()
