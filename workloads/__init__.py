"""Seeded synthetic inputs shared by the tests, bench.py and the oracle harness.

This module holds NO arithmetic of the lattice Boltzmann method: it only
produces the macroscopic fields of the paper's workloads, counter-based random
numbers, relaxation-rate vectors and the interface enumerations.  Both the
CUDA path (through the Python binding) and the CPU oracle (through tests) are
fed from here; neither side imports the other.

Workloads:
  * Taylor-Green vortex, eq:TGA_init, u0 = 0.25 (paper) or
    0.05 (parity), extruded along z for 3D; an (x,z)-plane variant exposes
    wrong slab planes in halo tests.
  * Circular dam break scaled to the grid.
  * Seeded noise U(-1,1) from splitmix64 of (seed, global cell index, i), so
    every rank, every decomposition and the oracle see identical fields.
"""
from __future__ import annotations

import math

import numpy as np

# ---- interface enumerations (mirrors include/lbm.h) ------------------------
D2Q9, D3Q19, D3Q27 = 0, 1, 2
STENCILS = {"D2Q9": D2Q9, "D3Q19": D3Q19, "D3Q27": D3Q27}
Q_OF = {D2Q9: 9, D3Q19: 19, D3Q27: 27}
DIM_OF = {D2Q9: 2, D3Q19: 3, D3Q27: 3}

POPULATION, RAW, CENTRAL, CUMULANT, RAW_WO = 0, 1, 2, 3, 4
SPACES = {"POPULATION": POPULATION, "RAW": RAW, "CENTRAL": CENTRAL, "CUMULANT": CUMULANT}
EQ_ABSOLUTE, EQ_DELTA, EQ_SWE, EQ_DISCRETE, EQ_DISCRETE_DELTA, EQ_ABSOLUTE_F0 = 0, 1, 2, 3, 4, 5
PERIODIC, NOSLIP = 0, 1

SEED = 221102435

# Basis-index groups of the documented bases (include/lbm.h, R2).
# conserved: order 0/1 polynomials; the rest keyed by the rate symbol.
RATE_GROUPS = {
    D2Q9: {
        "conserved": [0, 1, 2],
        "s": [3, 4],
        "b": [5],
        "3": [6, 7],
        "4": [8],
    },
    D3Q27: {
        "conserved": [0, 1, 2, 3],
        "s": [4, 5, 6, 7, 8],
        "b": [9],
        "3": [10, 11, 12],
        "4": [13, 14, 15],
        "5": [16],
        "6": [17, 18],
        "7": [19],
        "8": [20, 21, 22],
        "9": [23, 24, 25],
        "10": [26],
    },
    D3Q19: {
        "conserved": [0, 1, 2, 3],
        "s": [4, 5, 6, 7, 8],
        "b": [9],
        "3": [10, 11, 12],
        "4": [13, 14, 15],
        "6": [16, 17],
        "7": [18],
    },
}

# Rate set P: distinct per group so every path is exercised.
RATE_SET_P = {"conserved": 1.0, "s": 1.6, "b": 1.2, "3": 1.4, "4": 1.5, "5": 1.3,
              "6": 1.1, "7": 1.25, "8": 1.35, "9": 1.45, "10": 1.15}


def rates_from_groups(stencil: int, values: dict) -> np.ndarray:
    q = Q_OF[stencil]
    r = np.full(q, np.nan)
    for g, idx in RATE_GROUPS[stencil].items():
        r[idx] = values.get(g, 1.0)
    assert not np.isnan(r).any()
    return r


def rate_set_p(stencil: int) -> np.ndarray:
    return rates_from_groups(stencil, RATE_SET_P)


def regularized_rates(stencil: int, omega_s: float) -> np.ndarray:
    """R- methods: every rate but the shear rate set to one."""
    return rates_from_groups(stencil, {"s": omega_s})


def wo_second_order(stencil: int) -> list:
    """Indices of the second-order polynomials of the WO-MRT basis (graded-lexicographic
    order, include/lbm.h LBM_SPACE_RAW_WO): D2Q9 x^2, xy, y^2; 3D x^2, xy, xz, y^2, yz, z^2."""
    return [3, 4, 5] if DIM_OF[stencil] == 2 else [4, 5, 6, 7, 8, 9]


def wo_regularized_rates(stencil: int, omega_s: float) -> np.ndarray:
    """R-WO-MRT: every second-order polynomial of the WO basis at omega_s (in that basis the
    x^2 - 1/3 ... polynomials carry shear AND bulk viscosity), every other rate one."""
    r = np.ones(Q_OF[stencil])
    r[wo_second_order(stencil)] = omega_s
    return r


def rates_random(stencil: int, seed: int = SEED, lo: float = 0.7, hi: float = 1.9) -> np.ndarray:
    """One distinct rate per polynomial (catches index/ordering slips)."""
    q = Q_OF[stencil]
    u = counter_uniform(seed ^ 0x5A5A, np.arange(q, dtype=np.uint64), 1)[:, 0]
    return lo + (hi - lo) * (u + 1.0) / 2.0


def omega_from_nu(nu: float) -> float:
    """nu = cs^2 (1/omega - 1/2), cs^2 = 1/3  (nu = 1/6 <=> omega = 1)."""
    return 1.0 / (3.0 * nu + 0.5)


# ---- counter-based generator ------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def counter_uniform(seed: int, cell_index: np.ndarray, q: int) -> np.ndarray:
    """U(-1, 1) for each (global cell index, population i); shape [n, q]."""
    cell_index = np.asarray(cell_index, dtype=np.uint64).reshape(-1, 1)
    i = np.arange(q, dtype=np.uint64).reshape(1, -1)
    key = splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    with np.errstate(over="ignore"):
        ctr = (cell_index << np.uint64(6)) | i
        z = splitmix64(ctr ^ key)
    mant = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)  # [0, 1)
    return 2.0 * mant - 1.0


def noise_field(seed: int, q: int, nx: int, ny: int, nz: int, z0: int = 0, nz_global: int | None = None):
    """Noise U(-1,1) with layout [q][nz][ny][nx] for the z-planes [z0, z0+nz)
    of a global (nx, ny, nz_global) lattice (global linear index x + nx(y + ny z))."""
    z = np.arange(z0, z0 + nz, dtype=np.uint64).reshape(-1, 1, 1)
    y = np.arange(ny, dtype=np.uint64).reshape(1, -1, 1)
    x = np.arange(nx, dtype=np.uint64).reshape(1, 1, -1)
    gidx = (x + np.uint64(nx) * (y + np.uint64(ny) * z)).reshape(-1)
    u = counter_uniform(seed, gidx, q)  # [cells, q]
    return np.ascontiguousarray(u.T.reshape(q, nz, ny, nx))


# ---- macroscopic fields -----------------------------------------------------
def tgv_fields(nx: int, ny: int, nz: int, u0: float, nu: float = 1.0 / 6.0, t: float = 0.0,
               plane: str = "xy", z0: int = 0, nz_global: int | None = None):
    """Taylor-Green vortex, eq:TGA_init, at lattice node
    coordinates x = 0..L-1 (reading R10).  plane='xy' is the paper's field
    (extruded along z in 3D); plane='xz' puts the vortex in the (x, z) plane
    (reading R9).  For a non-square plane the wave numbers are k_a = 2 pi / n_a
    and the second velocity component is scaled by k_1/k_2 (divergence-free).
    Returns rho [nz][ny][nx], u [3][nz][ny][nx] (2D: nz = 1, u_z = 0)."""
    zs = np.arange(z0, z0 + nz, dtype=np.float64).reshape(-1, 1, 1)
    ys = np.arange(ny, dtype=np.float64).reshape(1, -1, 1)
    xs = np.arange(nx, dtype=np.float64).reshape(1, 1, -1)
    if plane == "xy":
        a, b, na, nb = xs, ys, nx, ny
    elif plane == "xz":
        nzg = nz_global if nz_global is not None else nz
        a, b, na, nb = xs, zs, nx, nzg
    else:
        raise ValueError(plane)
    ka, kb = 2 * math.pi / na, 2 * math.pi / nb
    k2 = 0.5 * (ka * ka + kb * kb)
    decay_u = math.exp(-2.0 * nu * k2 * t)
    decay_p = math.exp(-4.0 * nu * k2 * t)
    ua = u0 * np.cos(ka * a) * np.sin(kb * b) * decay_u
    ub = -u0 * (ka / kb) * np.sin(ka * a) * np.cos(kb * b) * decay_u
    rho = 1.0 - 0.75 * u0 * u0 * (np.cos(2 * ka * a) + np.cos(2 * kb * b)) * decay_p
    shape = (nz, ny, nx)
    rho = np.broadcast_to(rho, shape).astype(np.float64).copy()
    u = np.zeros((3,) + shape)
    u[0] = np.broadcast_to(ua, shape)
    if plane == "xy":
        u[1] = np.broadcast_to(ub, shape)
    else:
        u[2] = np.broadcast_to(ub, shape)
    return rho, u


def tgv_energy_ratio(nu: float, L: int, t: float) -> float:
    """E(t)/E0 = exp(-4 nu kappa^2 t), kappa = 2 pi / L (eq:TGA_kin_energy, reading R10)."""
    k = 2 * math.pi / L
    return math.exp(-4.0 * nu * k * k * t)


def dam_break_fields(nx: int, ny: int, radius: float, h_in: float, h_out: float, y0: int = 0,
                     ny_local: int | None = None):
    """Circular dam break: column of depth h_in and given
    radius (cells) centred in the domain, depth h_out elsewhere, u = 0.
    Returns h [1][ny_local][nx], u [3][1][ny_local][nx]."""
    nyl = ny if ny_local is None else ny_local
    ys = np.arange(y0, y0 + nyl, dtype=np.float64).reshape(-1, 1)
    xs = np.arange(nx, dtype=np.float64).reshape(1, -1)
    cx, cy = (nx - 1) / 2.0, (ny - 1) / 2.0
    r2 = (xs - cx) ** 2 + (ys - cy) ** 2
    h = np.where(r2 <= radius * radius, h_in, h_out).astype(np.float64)[None]
    return h, np.zeros((3,) + h.shape)


def swe_lattice_parameters(dx: float = 0.4, dt: float = 0.05, nu_phys: float = 1.0, g_phys: float = 9.81):
    """Lattice units of the dam break (reading R6): g_lat = g dt^2 / dx,
    nu_lat = nu dt / dx^2, omega_s = 1 / (3 nu_lat + 1/2) ~ 0.696."""
    g_lat = g_phys * dt * dt / dx
    nu_lat = nu_phys * dt / (dx * dx)
    return g_lat, nu_lat, omega_from_nu(nu_lat)
