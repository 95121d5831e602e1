#!/usr/bin/env python
"""Physics at the headline size: the C4 workload (D3Q27 cumulant, zc + absolute eq, fp64,
1024 x 1024 x 128, TGV extruded along z, u0 = 0.05, rate set P) run for N steps on the GPU;
kinetic energy and mass from the device diagnostics (lbm_get_diagnostics) against the
analytic decay E/E0 = exp(-4 nu k^2 t), k = 2 pi / 1024 (eq:TGA_kin_energy, reading R10),
nu from the shear rate (reading R3).

  python scripts/c4_physics.py [--steps 2000] [--every 500]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from paper_2211_02435_b200 import lbm as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--every", type=int, default=500)
    ap.add_argument("--shape", type=int, nargs=3, default=[1024, 1024, 128])
    args = ap.parse_args()
    st = W.D3Q27
    rates = W.rate_set_p(st)
    nu = (1.0 / rates[4] - 0.5) / 3.0  # shear group (reading R3)
    nx, ny, nz = args.shape
    rho, u = W.tgv_fields(nx, ny, nz, 0.05)
    out = {"shape": args.shape, "nu": nu, "samples": []}
    with L.Lattice(st, W.CUMULANT, W.EQ_ABSOLUTE, rates, tuple(args.shape), zero_centered=True) as lat:
        lat.init_macroscopic(rho, u)
        d0 = lat.get_diagnostics()
        t = 0
        while t < args.steps:
            lat.step(args.every)
            t += args.every
            d = lat.get_diagnostics()
            ratio = d["kinetic_energy"] / d0["kinetic_energy"]
            ref = W.tgv_energy_ratio(nu, nx, t)
            out["samples"].append({"t": t, "E_over_E0": ratio, "analytic": ref, "rel_dev": ratio / ref - 1,
                                   "mass_drift": d["mass"] / d0["mass"] - 1})
            print(f"t={t:6d}  E/E0={ratio:.9f}  analytic={ref:.9f}  rel.dev={ratio / ref - 1:+.2e}  "
                  f"mass drift={d['mass'] / d0['mass'] - 1:+.1e}", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
