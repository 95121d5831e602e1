"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The GPU runs the whole lattice (lbm_init_macroscopic from the analytic TGV / dam-break
fields, k fused steps); sampled output cells are compared with the oracle, which
recomputes each sample one by one on the (2k+1)^d neighbourhood that determines it
after k steps (its own equilibrium of the same analytic fields, then k pull+collide
steps; cells outside the dependency cone never reach the centre)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from gpu_helpers import F32_TOL, F64_TOL, gate_error, population_bound

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2211_02435_b200 import lbm as L  # noqa: E402

CONFIGS = {
    # name: stencil, space, eq, zc, precision, streaming, shape, steps
    "c4": (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, L.LBM_FP64, L.LBM_PULL, (1024, 1024, 128), 3),
    "c3": (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, L.LBM_FP64, L.LBM_AA, (384, 384, 384), 3),
    "c3_even": (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, L.LBM_FP64, L.LBM_AA, (384, 384, 384), 4),
    "c3_esoteric": (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, L.LBM_FP64, L.LBM_ESOTERIC_PULL, (384, 384, 384), 3),
    "c3_twist": (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, L.LBM_FP64, L.LBM_ESOTERIC_TWIST, (384, 384, 384), 4),
    "c4_aa": (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, L.LBM_FP64, L.LBM_AA, (1024, 1024, 128), 3),
    "c2_f64": (W.D3Q19, W.RAW, W.EQ_DELTA, 1, L.LBM_FP64, L.LBM_PULL, (256, 256, 256), 3),
    "c2_f32": (W.D3Q19, W.RAW, W.EQ_DELTA, 1, L.LBM_FP32, L.LBM_PULL, (256, 256, 256), 3),
    "c5": (W.D2Q9, W.CENTRAL, W.EQ_SWE, 0, L.LBM_FP64, L.LBM_PULL, (8192, 8192, 1), 3),
    "c3_push": (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, L.LBM_FP64, L.LBM_ESOTERIC_PUSH, (384, 384, 384), 3),
    "c5_zc": (W.D2Q9, W.CENTRAL, W.EQ_SWE, 1, L.LBM_FP64, L.LBM_PULL, (8192, 8192, 1), 4),
}


def fields(st, eq, shape):
    nx, ny, nz = shape
    if eq == W.EQ_SWE:
        h, u = W.dam_break_fields(nx, ny, nx * 2.5 / 40, 6.25, 1.25)
        return h, u
    if W.DIM_OF[st] == 2:
        return W.tgv_fields(nx, ny, 1, 0.05)
    return W.tgv_fields(nx, ny, nz, 0.05, plane="xz")


def samples(shape, n_random=24, seed=5):
    nx, ny, nz = shape
    rng = np.random.default_rng(seed)
    pts = [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (0, ny - 1, nz // 2), (nx - 1, 0, 0), (nx // 2, ny // 2, nz - 1),
           (1, 1, min(1, nz - 1))]
    for _ in range(n_random):
        pts.append((int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz))))
    return pts


@pytest.mark.parametrize("name", list(CONFIGS))
def test_fullsize_sampled_parity(name):
    st, space, eq, zc, prec, streaming, shape, k = CONFIGS[name]
    nx, ny, nz = shape
    d = W.DIM_OF[st]
    q = W.Q_OF[st]
    g = W.swe_lattice_parameters()[0] if eq == W.EQ_SWE else 0.0
    rates = W.regularized_rates(st, W.swe_lattice_parameters()[2]) if eq == W.EQ_SWE else W.rate_set_p(st)
    rho, u = fields(st, eq, shape)  # [nz][ny][nx] (2D: [1][ny][nx])
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, precision=prec, streaming=streaming,
                   swe_g=g) as lat:
        lat.init_macroscopic(rho, np.ascontiguousarray(u[:d]))
        lat.step(k)
        pts = samples(shape if d == 3 else (nx, ny, 1))
        idx = [x + nx * (y + ny * z) for (x, y, z) in pts]
        got = lat.get_cells(idx)  # [n][q]
    B = 2 * k + 1
    offs = np.arange(-k, k + 1)
    ref = np.empty_like(got)
    ref64 = np.empty_like(got)
    for s, (x, y, z) in enumerate(pts):
        xs = (x + offs) % nx
        ys = (y + offs) % ny
        if d == 3:
            zs = (z + offs) % nz
            r_box = rho[np.ix_(zs, ys, xs)]
            u_box = u[:, zs][:, :, ys][:, :, :, xs]
            bshape = (B, B, B)
        else:
            r_box = rho[0][np.ix_(ys, xs)][None]
            u_box = u[:, 0][:, ys][:, :, xs][:, None]
            bshape = (B, B, 1)
        feq = oracle.equilibrium(st, space, eq, zc, r_box.reshape(-1), u_box.reshape(3, -1).T, g=g)
        f0 = np.ascontiguousarray(feq.T.reshape((q,) + r_box.shape))
        if prec == L.LBM_FP32:
            f0 = f0.astype(np.float32).astype(np.float64)
        sim = oracle.Sim(st, space, eq, zc, rates, bshape, g=g)
        sim.set(f0)
        sim.step(k)
        out = sim.get()
        c = (k, k, k) if d == 3 else (0, k, k)
        ref[s] = out[(slice(None),) + c]
        if eq == W.EQ_SWE:  # the oracle's own fp64 error on the same box (reading R25)
            sim64 = oracle.Sim(st, space, eq, zc, rates, bshape, g=g, prec=oracle.DOUBLE)
            sim64.set(f0)
            sim64.step(k)
            ref64[s] = sim64.get()[(slice(None),) + c]
    tol = F32_TOL if prec == L.LBM_FP32 else F64_TOL
    if eq == W.EQ_SWE and zc:  # zero-centered shallow water: background f_eq(1, 0) (reading R33)
        f0 = oracle.equilibrium(st, space, eq, 0, np.ones(1), np.zeros((1, 3)), g=g)[0]
        got, ref, ref64, zc = got + f0, ref + f0, ref64 + f0, 0
    err = gate_error(st, got, ref, zc, cells_first=True)
    if eq == W.EQ_SWE:  # per-population gate at 10x the oracle's fp64 error, plus reading R12b
        disc = gate_error(st, ref64, ref, zc, cells_first=True)
        cell = gate_error(st, got, ref, zc, cells_first=True, norm="cell")
        print(f"{name}: per-population {err:.3e} (bound {population_bound(disc):.3e}), cell-normalised {cell:.3e}")
        assert cell < tol, cell
        tol = population_bound(disc)
    assert err < tol, err


def test_c5_fullsize_depth3_vs_depth2_long_run(monkeypatch):
    """Config 5 at its full size (8192^2 dam break) for 300 steps: three steps per sweep (the
    default) against two steps per sweep, to rounding on the cell-normalised metric (R12b), and
    the water volume conserved by both."""
    st, space, eq = W.D2Q9, W.CENTRAL, W.EQ_SWE
    g, nu, om = W.swe_lattice_parameters()
    rates = W.regularized_rates(st, om)
    shape = (8192, 8192, 1)
    h, u = fields(st, eq, shape)
    out = {}
    for depth in ("3", "2"):
        monkeypatch.setenv("LBM_TB_DEPTH", depth)
        with L.Lattice(st, space, eq, rates, shape, zero_centered=False, swe_g=g) as lat:
            assert lat.info().temporal_blocking == int(depth)
            lat.init_macroscopic(h, np.ascontiguousarray(u[:2]))
            m0 = lat.get_diagnostics()["mass"]
            lat.step(300)
            m1 = lat.get_diagnostics()["mass"]
            assert abs(m1 - m0) <= 1e-12 * m0
            idx = np.random.default_rng(3).integers(0, 8192 * 8192, 4096)
            out[depth] = lat.get_cells(idx)
    d = np.abs(out["3"] - out["2"]).max(axis=1) / np.abs(out["2"]).sum(axis=1)
    assert d.max() < 1e-13, d.max()
