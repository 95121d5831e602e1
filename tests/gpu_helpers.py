"""Shared helpers of the GPU parity tests: seeded initial states built by the
ORACLE (never by the CUDA path) and the parity metric (reading R12)."""
from __future__ import annotations

import numpy as np

import oracle
import workloads as W

F64_TOL = 1e-12  # BASELINE.json north_star: max relative population error, fp64
F32_TOL = 1e-5   # ... fp32


def q_of(st):
    return W.Q_OF[st]


def initial_state(st, space, eq, zc, shape, u0=0.05, noise=1e-3, plane="xz", seed=W.SEED, g=0.0,
                  z0=0, nz_global=None, dam=None):
    """Stored-form populations [q][nz][ny][nx] (2D: [q][1][ny][nx]): the oracle's
    equilibrium of a TGV (or dam-break) field plus seeded noise noise * w_i * U(-1,1)."""
    nx, ny, nz = shape
    q = q_of(st)
    xi, opp, w, M, Minv = oracle.tables(st)
    if dam is not None:
        rho, u = W.dam_break_fields(nx, ny, *dam)
        rho = rho.reshape(1, ny, nx)
        u = u.reshape(3, 1, ny, nx)
    elif W.DIM_OF[st] == 2:
        rho, u = W.tgv_fields(nx, ny, 1, u0, plane="xy")
    else:
        rho, u = W.tgv_fields(nx, ny, nz, u0, plane=plane, z0=z0, nz_global=nz_global)
    feq = oracle.equilibrium(st, space, eq, zc, rho.reshape(-1), u.reshape(3, -1).T, g=g)  # [cells, q]
    zz = nz if W.DIM_OF[st] == 3 else 1
    f = np.ascontiguousarray(feq.T.reshape(q, zz, ny, nx))
    if noise:
        U = W.noise_field(seed, q, nx, ny, zz, z0=z0)
        scale = w if dam is None else np.ones(q) * rho.mean()
        f = f + noise * scale[:, None, None, None] * U
    return f


def absolute(st, f, zc, cells_first=False):
    """Absolute populations f = stored + f0 (zero-centered) or stored.  Layout
    [q][...] (grids) or [cells][q] (cells_first, single-cell tests)."""
    if not zc:
        return f
    w = oracle.tables(st)[2]
    shape = (1, -1) if cells_first else (-1,) + (1,) * (f.ndim - 1)
    return f + w.reshape(shape)


def gate_error(st, f_gpu, f_ref, zc, cells_first=None, norm="population"):
    """Max over (x, i) of |f_gpu - f_ref| / |f_ref| on absolute populations (reading R12).
    norm='cell' divides by the cell's total sum_i |f_ref,i| instead (reading R12b: the
    shallow-water equilibrium has populations that approach zero, where a per-population
    relative error measures only the denominator)."""
    if cells_first is None:
        cells_first = f_gpu.ndim == 2
    a = absolute(st, f_gpu, zc, cells_first)
    b = absolute(st, f_ref, zc, cells_first)
    if norm == "cell":
        tot = np.abs(b).sum(axis=1 if cells_first else 0, keepdims=True)
        return float(np.max(np.abs(a - b) / tot))
    return float(np.max(np.abs(a - b) / np.abs(b)))


def field_error(st, f_gpu, f_ref):
    """Report-only: max |df_gpu - df_ref| / max |df_ref| (stored form)."""
    return float(np.max(np.abs(f_gpu - f_ref)) / max(np.max(np.abs(f_ref)), 1e-300))


def round_to(f, precision):
    from paper_2211_02435_b200 import lbm as L

    return f.astype(np.float32).astype(np.float64) if precision == L.LBM_FP32 else f


def oracle_run(st, space, eq, zc, rates, shape, f0, steps, bc=None, g=0.0):
    sim = oracle.Sim(st, space, eq, zc, rates, shape, bc=bc, g=g, prec=oracle.LONG_DOUBLE)
    sim.set(f0)
    sim.step(steps)
    return sim.get()


def oracle_fp64_discrepancy(st, space, eq, zc, rates, shape, f0, steps, ref, bc=None, g=0.0):
    """The oracle's own fp64 instantiation against its long-double reference `ref`, on the
    per-population gate metric: the error any correct fp64 implementation of the same run
    incurs (reading R25)."""
    sim = oracle.Sim(st, space, eq, zc, rates, shape, bc=bc, g=g, prec=oracle.DOUBLE)
    sim.set(f0)
    sim.step(steps)
    return gate_error(st, sim.get(), ref, zc)


def population_bound(disc):
    """Gate on the per-population metric where the parameters amplify round-off: the larger
    of the fp64 tolerance and 10x the oracle's own fp64-vs-long-double discrepancy."""
    return max(F64_TOL, 10.0 * disc)
