"""Builds liblbm.so (all kernels for sm_100a) in-tree with nvcc.

The kernel instantiations are split into one translation unit per
(stencil, precision, collision space, regime) so they compile in parallel;
the longest units (D3Q27 cumulant) are started first.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "liblbm.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -lineinfo keeps ncu's source view; the compressed fatbin keeps the many instantiations'
# line tables from quadrupling the library (10 -> 3 MB per D3Q27 unit)
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                  "-Xptxas", "-O3", "-Xfatbin", "-compress-all", "-diag-suppress", "177",
                  "-I", os.path.join(ROOT, "include")]

STENCILS = ["D2Q9", "D3Q19", "D3Q27"]
PRECS = {"f64": "double", "f32": "float"}
SPACES = ["POPULATION", "RAW", "CENTRAL", "CUMULANT"]
REGIMES = [0, 1, 2]  # absolute storage, zero-centered + delta eq, zero-centered + absolute eq


def units():
    out = []
    for st in STENCILS:
        for pr, real in PRECS.items():
            sps = SPACES + (["SWE", "SWEK"] if st == "D2Q9" else [])
            for sp in sps:
                for rg in REGIMES:
                    out.append((f"ops_{st}_{pr}_{sp}_r{rg}.o",
                                [f"-DLBM_STENCIL={st}", f"-DLBM_REAL={real}", f"-DLBM_PREC={pr}", f"-DLBM_SPACE={sp}",
                                 f"-DLBM_REGIME={rg}"],
                                "ops_inst.cu"))
    out.append(("runtime.o", [], "runtime.cu"))
    return out


def _headers():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + [
        os.path.join(ROOT, "include", "lbm.h")]


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + _headers() + [__file__])


def nvcc():
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return p


def build(jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    todo = []
    for obj, defs, src in units():
        o = os.path.join(OBJ, obj)
        s = os.path.join(CSRC, src)
        if _stale(o, s):
            todo.append([nvcc()] + NVFLAGS + defs + ["-c", s, "-o", o])
    jobs = jobs or max(1, os.cpu_count() or 1)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose:
            print(" ".join(cmd[-3:]), flush=True)
        return r

    # heaviest first: D3Q27 before D3Q19 before D2Q9, cumulant / central before the rest
    weight = {"D3Q27": 0, "D3Q19": 1, "D2Q9": 2}

    def key(cmd):
        o = os.path.basename(cmd[-1])
        st = next((k for k in weight if k in o), "D2Q9")
        return (weight[st], 0 if ("CUMULANT" in o or "CENTRAL" in o) else 1)

    todo.sort(key=key)
    with cf.ThreadPoolExecutor(jobs) as ex:
        list(ex.map(run, todo))
    objs = [os.path.join(OBJ, o) for o, _, _ in units()]
    if todo or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
