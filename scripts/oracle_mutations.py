#!/usr/bin/env python
"""Mutation check of the oracle's pins: plausible mistakes (a dropped term, a wrong sign,
index or operand) are injected one at a time into a copy of oracle/lbm_oracle.cpp, the
copy is built, and tests/test_oracle_pins.py must FAIL for every mutant.

  python scripts/oracle_mutations.py
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "lbm_oracle.cpp")

# (description, exact source snippet, replacement)
MUTANTS = [
    ("D3Q19 basis: drop the -2 in x^2y^2 - 2x^2z^2 + y^2z^2",
     "T(1, 2, 2, 0), T(-2, 2, 0, 2), T(1, 0, 2, 2)", "T(1, 2, 2, 0), T(-1, 2, 0, 2), T(1, 0, 2, 2)"),
    ("Maxwellian: cs2 = 1/2", "static const long double CS2 = 1.0L / 3.0L;", "static const long double CS2 = 1.0L / 2.0L;"),
    ("truncation at total degree 3", "if (i + j + k > 2) continue;", "if (i + j + k > 3) continue;"),
    ("series log: wrong sign", "R sgn = (n % 2 == 1) ? R(1) : R(-1);", "R sgn = R(1);"),
    # EQUIVALENT mutant, expected to survive: S^6 reaches degree <= 6 only through six first-order
    # factors, and the oracle takes the log of the CENTRAL moment series, whose first-order
    # coefficients vanish (kappa_100 = 0) - the n = 6 term is identically zero in every unforced
    # use; with a body force (R26) kappa_100 = -F/2 and the term is O((F/2 rho)^6) ~ 1e-24.
    ("series log: stop at n = 5 [equivalent]", "for (int n = 1; n <= 6; ++n) {\n    R sgn",
     "for (int n = 1; n <= 5; ++n) {\n    R sgn"),
    ("series exp: drop 1/n!", "for (int k = 0; k < 27; ++k) acc.c[k] += pw.c[k] / fact;",
     "for (int k = 0; k < 27; ++k) acc.c[k] += pw.c[k];"),
    ("e! factor: 2! -> 1", "static int efact(int e) { return e == 2 ? 2 : 1; }", "static int efact(int e) { return 1; }"),
    ("central moments: xi + u", "s += f[i] * ipow(R(m.xi[i][0]) - u[0], e[0])", "s += f[i] * ipow(R(m.xi[i][0]) + u[0], e[0])"),
    ("relaxation sign (raw)", "qs[p] = q0[p] + m.omega[p] * (qeq[p] - q0[p]) + (R(1) - m.omega[p] / R(2)) * qF[p];\n"
     "    matvec(q, m.Minv", "qs[p] = q0[p] - m.omega[p] * (qeq[p] - q0[p]) + (R(1) - m.omega[p] / R(2)) * qF[p];\n"
     "    matvec(q, m.Minv"),
    ("force: drop the (1 - w/2) factor (raw)", "+ (R(1) - m.omega[p] / R(2)) * qF[p];\n    matvec(q, m.Minv",
     "+ qF[p];\n    matvec(q, m.Minv"),
    ("force: no half-force velocity shift", "u[a] = (j[a] + R(half) * m.F[a] / R(2)) / rho;", "u[a] = j[a] / rho;"),
    ("force: 9 -> 3 in the Guo term", "R(3) * xF + R(9) * xu * xF - R(3) * uF", "R(3) * xF + R(3) * xu * xF - R(3) * uF"),
    ("cumulant eq: C_eq on xy instead of the diagonal",
     "(t.e[0] == 2 || t.e[1] == 2 || t.e[2] == 2)", "(t.e[0] == 1 || t.e[1] == 2 || t.e[2] == 2)"),
    ("zc: forget to add f0 for the absolute equilibrium",
     "fabs_[i] = (m.zc && !delta) ? fin[i] + m.w[i] : fin[i];", "fabs_[i] = fin[i];"),
    ("pull: push direction", "p[a] = pos[a] - s.m.xi[i][a];", "p[a] = pos[a] + s.m.xi[i][a];"),
    ("bounce-back: same slot instead of the opposite", "f[i] = src[(long long)s.m.opp[i] * N + c];",
     "f[i] = src[(long long)i * N + c];"),
    # a wall in the wrong place: the bounced population taken from the periodic image across the
    # wall (pinned by the closed-form channel flow, test_poiseuille_bounce_back_closed_form)
    ("bounce-back: opposite population of the periodic image instead of the own cell",
     "f[i] = src[(long long)s.m.opp[i] * N + c];",
     "f[i] = src[(long long)s.m.opp[i] * N + ((long long)p[2] * ny + p[1]) * nx + p[0]];"),
    ("SWE: printed -u.u/3 (the garble of Eq. 5.3)", "+ xu * xu / R(2) - uu / R(6));", "+ xu * xu / R(2) - uu / R(3));"),
    ("SWE cumulant: cs2 = g h", "const R cs2 = (m.eq == EQ_SWE) ? m.g * rho / R(2) : R(CS2);\n  // discrete",
     "const R cs2 = (m.eq == EQ_SWE) ? m.g * rho : R(CS2);\n  // discrete"),
    ("velocity: u = j (no division by rho)", "u[a] = (j[a] + R(half) * m.F[a] / R(2)) / rho;",
     "u[a] = (j[a] + R(half) * m.F[a] / R(2));"),
    ("cumulant force: F/2 instead of F on the first-order cumulants (R26)",
     "Cs.c[sidx(e100)] = C.c[sidx(e100)] + m.F[0];", "Cs.c[sidx(e100)] = C.c[sidx(e100)] + m.F[0] / R(2);"),
    ("cumulant force: source also on the cumulants of order >= 2 (R26)",
     "Cstar_poly[p] = Cpoly[p] + m.omega[p] * (ceq - Cpoly[p]);",
     "Cstar_poly[p] = Cpoly[p] + m.omega[p] * (ceq - Cpoly[p]) + m.F[0];"),
    ("He force: (xi + u) instead of (xi - u) (R27)", "cF += (R(m.xi[i][a]) - u[a]) * m.F[a];",
     "cF += (R(m.xi[i][a]) + u[a]) * m.F[a];"),
    ("He force: equilibrium without the background for zero-centered storage (R27)",
     "R fa = m.zc ? feq[i] + m.w[i] : feq[i];", "R fa = feq[i];"),
    ("discrete f_eq: 9/2 -> 3 on (xi.u)^2 (R29)", "R(3) * cu + R(9) * cu * cu / R(2) - R(3) * uu / R(2)",
     "R(3) * cu + R(3) * cu * cu - R(3) * uu / R(2)"),
    ("discrete f_eq: cumulant method falls back to the continuous C_eq (R29)",
     "ceq += R(t.c) * Cd.c[sidx(t.e)];\n        continue;", "(void)Cd;"),
    ("stencil order: swap (1,1) and (-1,-1) in-plane", "{1, 1}, {-1, -1}, {1, -1}, {-1, 1}};",
     "{-1, -1}, {1, 1}, {1, -1}, {-1, 1}};"),
    # the bulk rate (reading R3) acting on a wrong polynomial: pinned by the acoustic attenuation
    ("D2Q9: bulk rate on x^2 - y^2, shear rate on x^2 + y^2 (rows swapped)",
     "    B.push_back(P({T(1, 2, 0, 0), T(-1, 0, 2, 0)}));\n    B.push_back(P({T(1, 2, 0, 0), T(1, 0, 2, 0)}));",
     "    B.push_back(P({T(1, 2, 0, 0), T(1, 0, 2, 0)}));\n    B.push_back(P({T(1, 2, 0, 0), T(-1, 0, 2, 0)}));"),
    ("3D: bulk rate on x^2 - z^2, shear rate on x^2 + y^2 + z^2 (rows swapped)",
     "B.push_back(P({T(1, 2, 0, 0), T(-1, 0, 0, 2)}));                   // 8  x^2 - z^2\n"
     "  B.push_back(P({T(1, 2, 0, 0), T(1, 0, 2, 0), T(1, 0, 0, 2)}));     // 9  x^2 + y^2 + z^2",
     "B.push_back(P({T(1, 2, 0, 0), T(1, 0, 2, 0), T(1, 0, 0, 2)}));     // 8\n"
     "  B.push_back(P({T(1, 2, 0, 0), T(-1, 0, 0, 2)}));                   // 9"),
    # invisible to isotropy and to the incompressible TGV / shear-wave / Poiseuille pins
    ("bulk polynomial relaxed with the shear rate (omega_b ignored)",
     "    for (int i = 0; i < q; ++i) m.omega[i] = R(rates[i]);",
     "    for (int i = 0; i < q; ++i) m.omega[i] = R(rates[i]);\n"
     "    m.omega[stencil == ST_D2Q9 ? 5 : 9] = m.omega[stencil == ST_D2Q9 ? 4 : 7];"),
    # WO-MRT basis (reading R31)
    ("WO-MRT: unweighted Gram-Schmidt inner product (R31)",
     "num += m.w[i] * V[k * q + i] * P[j * q + i];\n        den += m.w[i] * P[j * q + i] * P[j * q + i];",
     "num += V[k * q + i] * P[j * q + i];\n        den += P[j * q + i] * P[j * q + i];"),
    ("WO-MRT: monomials in ascending instead of descending lexicographic order (R31)",
     "for (int a = 2; a >= 0; --a)\n      for (int b = 2; b >= 0; --b)",
     "for (int a = 0; a <= 2; ++a)\n      for (int b = 0; b <= 2; ++b)"),
    ("WO-MRT: subtracts cf times the monomial x^(e_j) instead of the orthogonalised p_j (R31)",
     "for (int i = 0; i < q; ++i) P[k * q + i] -= cf * P[j * q + i];",
     "for (int i = 0; i < q; ++i) P[k * q + i] -= cf * V[j * q + i];"),
    # zero-centered shallow water (reading R33)
    ("zc shallow water: background left at the lattice weights instead of f_eq(1, 0) (R33)",
     "const bool ok = equilibrium_cell(m, R(1), u0, m.w.data());", "const bool ok = true;"),
    ("zc shallow water: Zhou equilibrium not shifted by the background (R33)",
     "    if (m.zc)\n      for (int i = 0; i < q; ++i) f[i] -= m.w[i];\n    return true;",
     "    return true;"),
]


def main():
    src = open(SRC).read()
    tmp = tempfile.mkdtemp(prefix="oracle_mut_")
    gomp = subprocess.run(["g++", "-print-file-name=libgomp.so"], capture_output=True, text=True).stdout.strip()
    survived = []
    only = sys.argv[1:]  # optional substrings: run the matching mutants only
    for desc, old, new in MUTANTS:
        if only and not any(o in desc for o in only):
            continue
        if src.count(old) < 1:
            print(f"!! snippet not found: {desc}")
            survived.append(desc)
            continue
        mut = src.replace(old, new, 1)
        cpp = os.path.join(tmp, "m.cpp")
        so = os.path.join(tmp, "libm.so")
        open(cpp, "w").write(mut)
        r = subprocess.run(f"g++ -std=c++17 -O2 -ffp-contract=off -fopenmp -fPIC -c {cpp} -o {tmp}/m.o && "
                           f"g++ -shared -o {so} {tmp}/m.o -L{os.path.dirname(gomp)} -lgomp",
                           shell=True, capture_output=True, text=True)
        if r.returncode != 0:
            print(f"!! build failed: {desc}\n{r.stderr[-500:]}")
            survived.append(desc)
            continue
        env = dict(os.environ, LBM_ORACLE_LIB=so)
        t = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            os.path.join(ROOT, "tests", "test_oracle_pins.py")], env=env, capture_output=True,
                           text=True, cwd=ROOT, timeout=900)
        killed = t.returncode != 0
        first = [ln for ln in t.stdout.splitlines() if ln.startswith("FAILED")][:1]
        print(f"{'KILLED ' if killed else 'SURVIVED'}  {desc}  {first[0] if first else ''}", flush=True)
        if not killed and "[equivalent]" not in desc:
            survived.append(desc)
    shutil.rmtree(tmp, ignore_errors=True)
    run = [m for m in MUTANTS if not only or any(o in m[0] for o in only)]
    n_eq = sum("[equivalent]" in m[0] for m in run)
    print(f"{len(run) - n_eq - len(survived)}/{len(run) - n_eq} non-equivalent mutants killed "
          f"({n_eq} equivalent mutant(s) listed for the record)")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
