#!/usr/bin/env python
"""Circular dam break with the two shallow-water LBMs of the paper (
PAPER.md:1039-1077): central-moment method with Zhou's equilibrium (de Rosis) and the
cumulant method with the Maxwellian at cs2 = g h / 2 (Venturi).

Setup (reading R6): 40 m x 40 m periodic domain, 100 x 100 cells
(dx = 0.4 m), dt = 0.05 s, water column of radius 2.5 m and height 2.5 m at the centre,
0.5 m elsewhere, nu = 1 m^2/s => omega_s = 0.6957; every other rate one ("regularized").
Lattice units: h_lat = h / dx, g_lat = g dt^2 / dx.  Reports the water depth along the
cross-section y = 20 m at t = 1, 2, 3 s (Fig. 5) plus conservation and symmetry checks.

  python scripts/dam_break.py [--n 100] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_2211_02435_b200 import lbm as L  # noqa: E402


def run(space, n, dx, dt, times):
    g, nu, om = W.swe_lattice_parameters(dx=dx, dt=dt)
    st = W.D2Q9
    rates = W.regularized_rates(st, om)
    radius = 2.5 / dx
    h0, u0 = W.dam_break_fields(n, n, radius, 2.5 / dx, 0.5 / dx)
    out = {"omega_s": om, "g_lat": g, "profiles": {}, "min_h": {}, "mass": []}
    with L.Lattice(st, space, W.EQ_SWE, rates, (n, n, 1), zero_centered=False, swe_g=g) as lat:
        lat.init_macroscopic(h0, np.ascontiguousarray(u0[:2]))
        m0 = lat.get_diagnostics()["mass"]
        t_done = 0
        for t in times:
            steps = int(round(t / dt))
            lat.step(steps - t_done)
            t_done = steps
            h, u = lat.get_macroscopic()
            h = h[0]  # [y][x]
            # y = 20 m lies between rows n/2 - 1 and n/2 (cell centres at (i + 1/2) dx)
            prof = 0.5 * (h[n // 2 - 1] + h[n // 2]) * dx
            out["profiles"][f"{t:g}"] = prof.tolist()
            out["min_h"][f"{t:g}"] = float(prof.min())
            d = lat.get_diagnostics()
            out["mass"].append(d["mass"] / m0 - 1)
            sym = max(np.abs(h - h.T).max(), np.abs(h - h[::-1]).max(), np.abs(h - h[:, ::-1]).max())
            out.setdefault("symmetry_err", {})[f"{t:g}"] = float(sym)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1", "dam_break.json"))
    args = ap.parse_args()
    dx, dt = 40.0 / args.n, 0.05
    times = [1.0, 2.0, 3.0]
    res = {"setup": {"n": args.n, "dx_m": dx, "dt_s": dt, "times_s": times}}
    for name, space in (("CM", W.CENTRAL), ("K", W.CUMULANT)):
        r = run(space, args.n, dx, dt, times)
        res[name] = r
        print(f"{name}: omega_s = {r['omega_s']:.6f}; min depth on y = 20 m: " +
              ", ".join(f"t={t}: {v:.4f} m" for t, v in r["min_h"].items()) +
              f"; mass drift {max(abs(m) for m in r['mass']):.1e}; symmetry {max(r['symmetry_err'].values()):.1e}")
    d2 = res["K"]["min_h"]["2"] - res["CM"]["min_h"]["2"]
    res["K_minus_CM_trough_at_2s_m"] = d2
    print(f"trough depth K - CM at t = 2 s: {d2:+.4f} m (paper: K visibly deeper trough, PAPER.md:1067-1068)")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
