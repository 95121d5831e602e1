"""Auxiliary subsystems on the GPU: checkpoint/restart through the canonical state
(across streaming patterns), failure detection during runs, fp32 in-place patterns."""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W
from gpu_helpers import initial_state

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2211_02435_b200 import lbm as L  # noqa: E402


def test_checkpoint_restart_across_patterns(tmp_path):
    """Saving after 11 steps and continuing 6 more equals 17 uninterrupted steps bitwise, also
    when the checkpoint is written by an AA run and resumed by Esoteric Pull / pull runs."""
    st, space, eq, zc = W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1
    shape = (21, 10, 12)
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(17)
        ref = lat.get_populations()
    ck = tmp_path / "ck.npz"
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, streaming=L.LBM_AA) as lat:
        lat.set_populations(f0)
        lat.step(11)
        lat.save(ck)
    for streaming in (L.LBM_PULL, L.LBM_AA, L.LBM_ESOTERIC_PULL, L.LBM_ESOTERIC_TWIST):
        with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, streaming=streaming) as lat:
            assert lat.load(ck) == 11
            assert lat.info().steps_done == 11  # lbm_set_steps restores the counter
            lat.step(6)
            assert lat.info().steps_done == 17
            np.testing.assert_array_equal(lat.get_populations(), ref)
    with L.Lattice(st, W.CENTRAL, eq, rates, shape, zero_centered=zc) as lat:
        with pytest.raises(ValueError):
            lat.load(ck)


def test_run_detects_non_finite_state():
    st = W.D2Q9
    shape = (16, 12, 1)
    f0 = initial_state(st, W.RAW, W.EQ_DELTA, 1, shape)
    f0[4, 0, 5, 7] = np.inf
    seen = []
    with L.Lattice(st, W.RAW, W.EQ_DELTA, W.rate_set_p(st), shape) as lat:
        lat.set_populations(f0)
        with pytest.raises(L.LbmError) as e:
            lat.run(10, check_every=2, callback=lambda l, s: seen.append(s), every=1)
        assert e.value.status == L.LBM_ENUMERIC
        assert "step 2" in str(e.value)
    assert seen == [1]


def test_run_intervals_count_from_the_call():
    """run(n, check_every, every) with intervals that are not multiples of each other, on a
    context that already advanced: the probe and the callback fire at every multiple of their
    own interval counted from the start of the call."""
    st = W.D2Q9
    shape = (16, 12, 1)
    f0 = initial_state(st, W.RAW, W.EQ_DELTA, 1, shape)
    seen, probes = [], []
    with L.Lattice(st, W.RAW, W.EQ_DELTA, W.rate_set_p(st), shape) as lat:
        lat.set_populations(f0)
        lat.step(1)
        orig = lat.check_finite
        lat.check_finite = lambda: (probes.append(lat.info().steps_done), orig())[1]
        lat.run(12, check_every=2, callback=lambda l, s: seen.append(s), every=3)
    assert probes == [3, 5, 7, 9, 11, 13]
    assert seen == [4, 7, 10, 13]
    # the same run in one go or in the run() chunks: identical state
    with L.Lattice(st, W.RAW, W.EQ_DELTA, W.rate_set_p(st), shape) as a, \
            L.Lattice(st, W.RAW, W.EQ_DELTA, W.rate_set_p(st), shape) as b:
        a.set_populations(f0)
        b.set_populations(f0)
        a.step(13)
        b.step(1)
        b.run(12, check_every=5, every=7)
        assert np.array_equal(a.get_populations(), b.get_populations())


@pytest.mark.parametrize("st", [W.D2Q9, W.D3Q19, W.D3Q27])
def test_fp32_in_place_patterns_equal_pull(st):
    shape = (20, 12, 1) if st == W.D2Q9 else (20, 10, 12)
    space, eq, zc = W.CENTRAL, W.EQ_ABSOLUTE, 1
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape).astype(np.float32).astype(np.float64)
    outs = []
    for streaming in (L.LBM_PULL, L.LBM_AA, L.LBM_ESOTERIC_PULL, L.LBM_ESOTERIC_TWIST, L.LBM_ESOTERIC_PUSH):
        with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, precision=L.LBM_FP32,
                       streaming=streaming) as lat:
            lat.set_populations(f0)
            lat.step(7)
            outs.append(lat.get_populations())
    for other in outs[1:]:
        np.testing.assert_array_equal(outs[0], other)


@pytest.mark.parametrize("st,space,eq,streaming", [
    (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, L.LBM_PULL),
    (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, L.LBM_AA),
    (W.D3Q19, W.RAW, W.EQ_DELTA, L.LBM_PULL),
    (W.D3Q27, W.CENTRAL, W.EQ_DISCRETE, L.LBM_ESOTERIC_TWIST),
])
def test_gpu_tgv_second_order_convergence(st, space, eq, streaming):
    """Physics of the GPU path beyond the sizes the oracle reaches: the Taylor-Green decay
    E/E0 = exp(-4 nu kappa^2 t) (eq:TGA_kin_energy) at L = 32, 64, 128 (extruded along z,
    4 planes) converges at second order under diffusive scaling (error ratio ~4)."""
    nu = 0.05
    om = W.omega_from_nu(nu)
    rates = W.regularized_rates(st, om)
    errs = []
    for Ln in (32, 64, 128):
        shape = (Ln, Ln, 4)
        k = 2 * np.pi / Ln
        steps = int(round(np.log(2) / (4 * nu * k * k)))
        rho, u = W.tgv_fields(Ln, Ln, 4, 0.05 * 64 / Ln)
        with L.Lattice(st, space, eq, rates, shape, zero_centered=True, streaming=streaming) as lat:
            lat.init_macroscopic(rho, u)
            r0, u0 = lat.get_macroscopic()
            e0 = 0.5 * (r0 * (u0 ** 2).sum(0)).sum()
            lat.step(steps)
            r1, u1 = lat.get_macroscopic()
            e1 = 0.5 * (r1 * (u1 ** 2).sum(0)).sum()
        errs.append(abs(e1 / e0 / W.tgv_energy_ratio(nu, Ln, steps) - 1))
    assert errs[-1] < 5e-3, errs
    for a, b in zip(errs, errs[1:]):
        assert 3.5 < a / b < 4.5, errs


@pytest.mark.parametrize("st,space", [(W.D3Q27, W.CUMULANT), (W.D3Q19, W.RAW), (W.D2Q9, W.CENTRAL),
                                      (W.D3Q27, W.POPULATION)])
def test_background_density_scaling_bitwise(st, space):
    """rho0 is a unit choice (reading R21; pinned on the oracle by
    test_background_density_is_a_unit_choice): on absolute storage the device update is
    homogeneous of degree one, and scaling by 2 is exact in fp64, so 10 steps of 2 f equal
    2 x (10 steps of f) bitwise — a run at background density 2 is the rho0 = 1 run in other
    units."""
    shape = (20, 12, 1) if st == W.D2Q9 else (20, 10, 12)
    rates = [1.3] if space == W.POPULATION else W.rate_set_p(st)
    f0 = initial_state(st, space, W.EQ_ABSOLUTE, 0, shape)
    outs = []
    for lam in (1.0, 2.0):
        with L.Lattice(st, space, W.EQ_ABSOLUTE, rates, shape, zero_centered=False) as lat:
            lat.set_populations(lam * f0)
            lat.step(10)
            outs.append(lat.get_populations())
    np.testing.assert_array_equal(outs[1], 2.0 * outs[0])


@pytest.mark.parametrize("space", [W.CENTRAL, W.CUMULANT])
def test_swe_depth_scaling_bitwise(space):
    """h0 is a gravity rescaling (test_swe_background_depth_is_a_gravity_rescaling): the
    shallow-water run of 2 f at gravity g equals 2 x the run of f at gravity 2 g, bitwise."""
    st, shape = W.D2Q9, (24, 16, 1)
    g = 0.0613125
    f0 = initial_state(st, space, W.EQ_SWE, 0, shape, g=2 * g, noise=0.0, dam=(6.0, 4.0, 1.25))
    with L.Lattice(st, space, W.EQ_SWE, W.rate_set_p(st), shape, zero_centered=False, swe_g=2 * g) as lat:
        lat.set_populations(f0)
        lat.step(10)
        a = lat.get_populations()
    with L.Lattice(st, space, W.EQ_SWE, W.rate_set_p(st), shape, zero_centered=False, swe_g=g) as lat:
        lat.set_populations(2 * f0)
        lat.step(10)
        b = lat.get_populations()
    np.testing.assert_array_equal(b, 2 * a)


@pytest.mark.parametrize("st,space,tau,model,streaming", [
    (W.D2Q9, W.POPULATION, 1.0, 0, L.LBM_PULL),
    (W.D2Q9, W.CUMULANT, 0.875, 1, L.LBM_PULL),
    (W.D3Q19, W.RAW, 0.8, 0, L.LBM_AA),
    (W.D3Q27, W.CUMULANT, 1.1, 0, L.LBM_PULL),
    (W.D3Q27, W.CENTRAL, 0.65, 1, L.LBM_AA),
])
def test_gpu_poiseuille_bounce_back_closed_form(st, space, tau, model, streaming):
    """The device path (walls + body force, pull and AA in place) against the closed-form
    steady channel flow of half-way bounce-back (tests/test_oracle_pins.py
    test_poiseuille_bounce_back_closed_form: u_x(y) = F / (2 nu) [(y + 1/2)(H - 1/2 - y) +
    (16 Lambda - 3) / 12]) — a pin of reading R18 independent of the oracle."""
    nx, ny, Fx = 32, 8, 1e-6
    nz = 1 if W.DIM_OF[st] == 2 else 4
    nu = (tau - 0.5) / 3
    rates = [1 / tau] if space == W.POPULATION else W.regularized_rates(st, 1 / tau)
    lam = (tau - 0.5) * ((tau - 0.5) if space == W.POPULATION else 0.5)
    bc = [[0, 0], [L.LBM_BC_NOSLIP] * 2, [0, 0]]
    eq = W.EQ_ABSOLUTE if space == W.CUMULANT else W.EQ_DELTA
    with L.Lattice(st, space, eq, rates, (nx, ny, nz), zero_centered=True, bc=bc, streaming=streaming) as lat:
        lat.set_populations(np.zeros((W.Q_OF[st], nz, ny, nx)))
        lat.set_force([Fx, 0, 0], model=model)
        lat.step(30000)
        _, u = lat.get_macroscopic()
    y = np.arange(ny)
    ref = Fx / (2 * nu) * ((y + 0.5) * (ny - 0.5 - y) + (16 * lam - 3) / 12)
    ux = u[0].reshape(nz, ny, nx)
    assert np.abs(ux - ref[None, :, None]).max() < 1e-9 * ref.max()
    assert np.abs(u[1:]).max() < 1e-12 * ref.max()
