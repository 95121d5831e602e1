#!/usr/bin/env python
"""Table 3 of the paper on B200: round-off plateaus of the
Taylor-Green vortex energy for D3Q27 methods and storage/equilibrium formats.

Setup: TGV eq:TGA_init with u0 = 0.25, nu = 1/6 (omega = 1),
kappa = 2 pi / L, L = 256, periodic L^3 box (the 2D field extruded along z,
reading R9); 200 000 time steps; E(t)/E0 with E = sum rho |u|^2 / 2 over the
lattice nodes (eq:TGA_kin_energy).  Methods: SRT, R-WO-MRT (the weighted-orthogonal raw
basis, LBM_SPACE_RAW_WO, reading R31), R-RAW (the raw basis of reading R2), R-CM, R-K;
formats: absolute storage; zero-centered + absolute equilibrium written literally, f0 added
to the populations before the transform (LBM_EQ_ABSOLUTE_F0, reading R30: the paper's
"zc + f^eq"); zero-centered + absolute equilibrium with the background added in moment space
(LBM_EQ_ABSOLUTE, our default); zero-centered + delta equilibrium (admissible ones only,
PAPER.md:545-547).

  python scripts/table3_roundoff.py [--L 256] [--steps 200000] [--every 2000] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_2211_02435_b200 import lbm as L  # noqa: E402

# paper's Table 3: E/E0 after 200 000 steps
PAPER = {
    ("SRT", "abs"): 1.9e-26, ("SRT", "zc+delta"): 5.4e-33,
    ("R-WO-MRT", "abs"): 1.7e-29, ("R-WO-MRT", "zc+eq"): 4.4e-31, ("R-WO-MRT", "zc+delta"): 6.1e-33,
    ("R-CM", "abs"): 2.4e-29, ("R-CM", "zc+eq"): 2.7e-33, ("R-CM", "zc+delta"): 1.7e-34,
    ("R-K", "abs"): 9.1e-27, ("R-K", "zc+eq"): 1.1e-32,
}

METHODS = [("SRT", W.POPULATION), ("R-WO-MRT", W.RAW_WO), ("R-RAW", W.RAW), ("R-CM", W.CENTRAL),
           ("R-K", W.CUMULANT)]
# "zc+eq" is the paper's zc + f^eq column: the literal form (f0 added to the populations)
FORMATS = {"abs": (W.EQ_ABSOLUTE, 0), "zc+eq": (W.EQ_ABSOLUTE_F0, 1), "zc+eq(moments)": (W.EQ_ABSOLUTE, 1),
           "zc+delta": (W.EQ_DELTA, 1)}


def run_one(space, eq, zc, L_, steps, every, u0=0.25, nu=1.0 / 6.0):
    st = W.D3Q27
    om = W.omega_from_nu(nu)
    if space == W.POPULATION:
        rates = [om]
    elif space == W.RAW_WO:
        rates = W.wo_regularized_rates(st, om)
    else:
        rates = W.regularized_rates(st, om)
    rho, u = W.tgv_fields(L_, L_, L_, u0)
    with L.Lattice(st, space, eq, rates, (L_, L_, L_), zero_centered=zc) as lat:
        lat.init_macroscopic(rho, u)
        e0 = lat.get_diagnostics()["kinetic_energy"]
        series = [(0, 1.0)]
        t0 = time.perf_counter()
        done = 0
        while done < steps:
            k = min(every, steps - done)
            lat.step(k)
            done += k
            series.append((done, lat.get_diagnostics()["kinetic_energy"] / e0))
        lat.sync()
        dt = time.perf_counter() - t0
        rs = lat.info().rate_specialization
    return series, dt, rs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=256)
    ap.add_argument("--steps", type=int, default=200000)
    ap.add_argument("--every", type=int, default=2000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2", "table3_roundoff.json"))
    ap.add_argument("--only", default=None, help="comma list of METHOD:FORMAT")
    args = ap.parse_args()
    nu = 1.0 / 6.0
    k = 2 * math.pi / args.L
    results = []
    for name, space in METHODS:
        for fmt, (eq, zc) in FORMATS.items():
            if space == W.CUMULANT and eq == W.EQ_DELTA:
                continue  # inadmissible
            if args.only and f"{name}:{fmt}" not in args.only.split(","):
                continue
            series, dt, rs = run_one(space, eq, zc, args.L, args.steps, args.every)
            final = series[-1][1]
            # accuracy against the analytic decay while it is resolvable (t <= 20 000)
            dev = max(abs(v / math.exp(-4 * nu * k * k * t) - 1) for t, v in series if 0 < t <= 20000)
            row = {"method": name, "format": fmt, "E_over_E0_final": final, "steps": args.steps, "L": args.L,
                   "paper": PAPER.get((name, fmt)), "max_rel_dev_analytic_t_le_20000": dev,
                   "seconds": dt, "mlups": args.L ** 3 * args.steps / dt / 1e6, "rate_specialization": rs,
                   "series": series}
            results.append(row)
            print(f"{name:9s} {fmt:9s} E/E0 = {final:.3e}  (paper {PAPER.get((name, fmt))})  "
                  f"dev<=2e4: {dev:.2e}  {dt:.1f} s", flush=True)
    analytic = math.exp(-4 * nu * k * k * args.steps)
    out = {"analytic_E_over_E0_final": analytic, "results": results,
           "setup": "D3Q27 TGV u0=0.25 nu=1/6 L^3 periodic, fp64, B200, pull streaming"}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"analytic E/E0 at t = {args.steps}: {analytic:.3e}")


if __name__ == "__main__":
    main()
