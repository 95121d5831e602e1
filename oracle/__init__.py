"""ctypes wrapper of the CPU oracle (oracle/lbm_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py — never by the product
package paper_2211_02435_b200/.  It shares no code with the CUDA path.

Parity-status of each oracle function is listed in DESIGN.md §"Oracle pins";
every function here is pinned by tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

LONG_DOUBLE, DOUBLE = 1, 0


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.environ.get("LBM_ORACLE_LIB")  # mutation checks (scripts/oracle_mutations.py)
        if not path:
            path = os.path.join(_HERE, "liboracle.so")
            src = os.path.join(_HERE, "lbm_oracle.cpp")
            if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
                build()
        L = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        L.oracle_tables.argtypes = [ctypes.c_int, ip, ip, ip, dp, dp, dp]
        L.oracle_collide.argtypes = [ctypes.c_int] * 4 + [dp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                                          dp, dp, ctypes.c_longlong]
        L.oracle_equilibrium.argtypes = [ctypes.c_int] * 4 + [ctypes.c_double, dp, dp, dp, ctypes.c_longlong]
        L.oracle_central_and_cumulants.argtypes = [ctypes.c_int, dp, ctypes.c_longlong, dp, dp, dp, dp]
        L.oracle_cumulant_roundtrip.argtypes = [dp, ctypes.c_double, dp]
        L.oracle_sim_create.restype = ctypes.c_void_p
        L.oracle_sim_create.argtypes = [ctypes.c_int] * 4 + [dp, ctypes.c_int, ctypes.c_double,
                                                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ip,
                                                             ctypes.c_int]
        L.oracle_sim_destroy.argtypes = [ctypes.c_void_p]
        L.oracle_sim_set.argtypes = [ctypes.c_void_p, dp]
        L.oracle_sim_get.argtypes = [ctypes.c_void_p, dp]
        L.oracle_sim_step.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.oracle_sim_macroscopic.argtypes = [ctypes.c_void_p, dp, dp]
        L.oracle_collide_forced.argtypes = [ctypes.c_int] * 4 + [dp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                                                 dp, dp, dp, ctypes.c_longlong]
        L.oracle_sim_set_force.argtypes = [ctypes.c_void_p, dp]
        L.oracle_collide_forced_model.argtypes = [ctypes.c_int] * 4 + [dp, ctypes.c_int, ctypes.c_double,
                                                                       ctypes.c_int, dp, ctypes.c_int, dp, dp,
                                                                       ctypes.c_longlong]
        L.oracle_sim_set_force_model.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.oracle_wo_basis.argtypes = [ctypes.c_int, dp, dp, ip]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _LIB = L
    return _LIB


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def tables(stencil: int):
    """(xi [q,3], opp [q], w [q], M [q,q], Minv [q,q]) as the oracle derives them."""
    q = ctypes.c_int()
    xi = np.zeros(27 * 3, np.int32)
    opp = np.zeros(27, np.int32)
    w = np.zeros(27)
    M = np.zeros(27 * 27)
    Minv = np.zeros(27 * 27)
    rc = lib().oracle_tables(stencil, ctypes.byref(q), _ip(xi), _ip(opp), _dp(w), _dp(M), _dp(Minv))
    assert rc == 0
    n = q.value
    return (xi[: 3 * n].reshape(n, 3).copy(), opp[:n].copy(), w[:n].copy(),
            M[: n * n].reshape(n, n).copy(), Minv[: n * n].reshape(n, n).copy())


GUO, HE = 0, 1  # force models (readings R23, R27)


def collide(stencil, space, eq, zc, rates, f_in, g=0.0, prec=LONG_DOUBLE, force=None, force_model=GUO):
    """Collision of independent cells; f_in [n, q] in stored form; optional uniform body
    force density force[3] (Guo forcing, reading R23, or He forcing, reading R27)."""
    f_in = np.ascontiguousarray(f_in, dtype=np.float64)
    out = np.empty_like(f_in)
    r = np.ascontiguousarray(rates, dtype=np.float64).reshape(-1)
    if force is not None:
        F = np.ascontiguousarray(np.asarray(force, dtype=np.float64).reshape(3))
        rc = lib().oracle_collide_forced_model(stencil, space, eq, int(zc), _dp(r), r.size, float(g), prec,
                                               _dp(F), int(force_model), _dp(f_in), _dp(out), f_in.shape[0])
    else:
        rc = lib().oracle_collide(stencil, space, eq, int(zc), _dp(r), r.size, float(g), prec, _dp(f_in),
                                  _dp(out), f_in.shape[0])
    if rc != 0:
        raise RuntimeError(f"oracle_collide failed ({rc})")
    return out


def equilibrium(stencil, space, eq, zc, rho, u, g=0.0):
    """f_eq per cell, stored form; rho [n], u [n, 3]  ->  [n, q]."""
    rho = np.ascontiguousarray(rho, dtype=np.float64).reshape(-1)
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1, 3)
    q = {0: 9, 1: 19, 2: 27}[stencil]
    out = np.empty((rho.size, q))
    rc = lib().oracle_equilibrium(stencil, space, eq, int(zc), float(g), _dp(rho), _dp(u), _dp(out), rho.size)
    if rc != 0:
        raise RuntimeError(f"oracle_equilibrium failed ({rc})")
    return out


def central_and_cumulants(stencil, f_abs):
    """Monomial central moments and rescaled cumulants (27 each, e = ex + 3ey + 9ez)."""
    f_abs = np.ascontiguousarray(f_abs, dtype=np.float64)
    n = f_abs.shape[0]
    k = np.empty((n, 27))
    C = np.empty((n, 27))
    rho = np.empty(n)
    u = np.empty((n, 3))
    lib().oracle_central_and_cumulants(stencil, _dp(f_abs), n, _dp(k), _dp(C), _dp(rho), _dp(u))
    return k, C, rho, u


def cumulant_roundtrip(kappa27, rho):
    k = np.ascontiguousarray(kappa27, dtype=np.float64)
    out = np.empty(27)
    lib().oracle_cumulant_roundtrip(_dp(k), float(rho), _dp(out))
    return out


class Sim:
    """Two-grid pull simulation; state [q][nz][ny][nx] in stored form."""

    def __init__(self, stencil, space, eq, zc, rates, shape, bc=None, g=0.0, prec=LONG_DOUBLE):
        nx, ny, nz = shape
        self.q = {0: 9, 1: 19, 2: 27}[stencil]
        self.shape = (self.q, nz, ny, nx)
        r = np.ascontiguousarray(rates, dtype=np.float64).reshape(-1)
        bca = np.zeros(6, np.int32) if bc is None else np.ascontiguousarray(np.asarray(bc, np.int32).reshape(6))
        self._h = lib().oracle_sim_create(stencil, space, eq, int(zc), _dp(r), r.size, float(g), nx, ny, nz,
                                          _ip(bca), prec)
        if not self._h:
            raise ValueError("oracle_sim_create rejected the method")

    def set(self, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        assert f.shape == self.shape
        lib().oracle_sim_set(self._h, _dp(f))

    def get(self):
        f = np.empty(self.shape)
        lib().oracle_sim_get(self._h, _dp(f))
        return f

    def step(self, n=1):
        lib().oracle_sim_step(self._h, int(n))

    def set_force(self, force, force_model=GUO):
        F = np.ascontiguousarray(np.asarray(force, dtype=np.float64).reshape(3))
        lib().oracle_sim_set_force(self._h, _dp(F))
        if lib().oracle_sim_set_force_model(self._h, int(force_model)) != 0:
            raise ValueError("unknown force model")

    def macroscopic(self):
        q, nz, ny, nx = self.shape
        rho = np.empty((nz, ny, nx))
        u = np.empty((3, nz, ny, nx))
        lib().oracle_sim_macroscopic(self._h, _dp(rho), _dp(u))
        return rho, u

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().oracle_sim_destroy(h)
            self._h = None


def max_threads() -> int:
    return lib().oracle_max_threads()


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle (torchrun exports OMP_NUM_THREADS=1 to every rank)."""
    lib().oracle_set_threads(int(n))


def wo_basis(stencil: int):
    """WO-MRT basis (reading R31) as the oracle builds it: (M [q,q] with M[k,i] = p_k(xi_i),
    G [q,q] monomial coefficients, mono [q,3] graded-lexicographic exponents)."""
    M = np.zeros(27 * 27)
    G = np.zeros(27 * 27)
    mono = np.zeros(27 * 3, np.int32)
    q = lib().oracle_wo_basis(stencil, _dp(M), _dp(G), _ip(mono))
    if q < 0:
        raise RuntimeError("oracle_wo_basis failed")
    return M[: q * q].reshape(q, q).copy(), G[: q * q].reshape(q, q).copy(), mono[: 3 * q].reshape(q, 3).copy()
