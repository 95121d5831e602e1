"""Pins of the CPU oracle against what the paper and the mathematics fix.

Nothing here compares the oracle with itself or with the CUDA path: every
expected value is a paper value (tests/golden/, cited), a closed form, a
textbook relation derived independently in this file (moment-cumulant
partition formula, textbook BGK equilibrium, Gaussian product distribution),
an invariant, or brute force on tiny inputs.
"""
from __future__ import annotations

import itertools
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
STENCILS = [W.D2Q9, W.D3Q19, W.D3Q27]
LINEAR_SPACES = [W.POPULATION, W.RAW, W.CENTRAL]
ALL_REGIMES = [(W.EQ_ABSOLUTE, 0), (W.EQ_DELTA, 1), (W.EQ_ABSOLUTE, 1)]


def admissible(space):
    """(eq, zc) pairs admissible for a space."""
    if space == W.CUMULANT:
        return [(W.EQ_ABSOLUTE, 0), (W.EQ_ABSOLUTE, 1)]
    return ALL_REGIMES


def rates_for(stencil, space, value=None, seed=7):
    if space == W.POPULATION:
        return np.array([1.3 if value is None else value])
    if value is not None:
        return np.full(W.Q_OF[stencil], float(value))
    return W.rates_random(stencil, seed=seed)


def random_cells(stencil, n, amp=2e-2, seed=3, umax=0.08):
    """Absolute populations near a random equilibrium-ish state (positive)."""
    xi, opp, w, M, Minv = oracle.tables(stencil)
    rng = np.random.default_rng(seed)
    rho = 1.0 + rng.uniform(-0.05, 0.05, n)
    u = rng.uniform(-umax, umax, (n, 3))
    if W.DIM_OF[stencil] == 2:
        u[:, 2] = 0
    f = textbook_feq(stencil, rho, u)
    f += amp * w * rng.uniform(-1, 1, f.shape)
    return f


def textbook_feq(stencil, rho, u):
    """Second-order Hermite equilibrium f_i = w_i rho (1 + 3 xi.u + 9/2 (xi.u)^2 - 3/2 u^2)
    (textbook, e.g. Krueger et al. 2017 eq. 3.54 — typed here independently)."""
    xi, opp, w, M, Minv = oracle.tables(stencil)
    cu = u @ xi.T
    uu = (u * u).sum(1, keepdims=True)
    return w * rho[:, None] * (1 + 3 * cu + 4.5 * cu * cu - 1.5 * uu)


def product_feq(stencil, rho, u):
    """Equilibrium whose central moments are the Gaussian's (u-independent):
    f = rho prod_a phi(xi_a, u_a), phi(0) = 1 - cs2 - u^2, phi(+-1) = (cs2 + u^2 +- u)/2.
    Typed here from the per-axis moment conditions (sum 1, mean u, var cs2)."""
    xi, opp, w, M, Minv = oracle.tables(stencil)
    d = W.DIM_OF[stencil]
    f = np.ones((rho.size, xi.shape[0])) * rho[:, None]
    for a in range(d):
        ua = u[:, a:a + 1]
        x = xi[None, :, a]
        phi = np.where(x == 0, 1 - 1 / 3 - ua * ua, (1 / 3 + ua * ua + x * ua) / 2)
        f = f * phi
    return f


# ---------------------------------------------------------------- stencils ---
def test_weights_golden():
    """f0 = M^{-1} m0 reduces to the lattice weights."""
    gold = {}
    for line in open(os.path.join(GOLDEN, "weights.txt")):
        if line.startswith("#") or not line.strip():
            continue
        st, n2, num, den = line.split()
        gold[(W.STENCILS[st], int(n2))] = int(num) / int(den)
    for st in STENCILS:
        xi, opp, w, M, Minv = oracle.tables(st)
        for i in range(len(w)):
            n2 = int((xi[i] ** 2).sum())
            assert w[i] == pytest.approx(gold[(st, n2)], abs=1e-16), (st, i)
        assert w.sum() == pytest.approx(1.0, abs=1e-15)


@pytest.mark.parametrize("st", STENCILS)
def test_stencil_convention(st):
    """xi_0 = 0; opposite pairs; slab-axis groups contiguous
    (interface convention of include/lbm.h)."""
    xi, opp, w, M, Minv = oracle.tables(st)
    q = W.Q_OF[st]
    assert xi.shape == (q, 3)
    assert (xi[0] == 0).all()
    assert len({tuple(v) for v in xi}) == q
    for i in range(q):
        assert (xi[opp[i]] == -xi[i]).all()
        assert opp[opp[i]] == i
    slab = 1 if st == W.D2Q9 else 2
    comp = xi[:, slab]
    n_up = int((comp == 1).sum())
    first_up = int(np.argmax(comp == 1))
    # +1 group contiguous, followed by the -1 group as its negation in the same order
    assert (comp[first_up:first_up + n_up] == 1).all()
    assert (comp[first_up + n_up:] == -1).all()
    for k in range(n_up):
        assert opp[first_up + k] == first_up + n_up + k
    assert n_up == {W.D2Q9: 3, W.D3Q19: 5, W.D3Q27: 9}[st]
    if st == W.D3Q19:
        assert (np.abs(xi).sum(1) <= 2).all()


def test_stencil_order_golden():
    """The full documented velocity order (tests/golden/stencil_order.txt, include/lbm.h)."""
    gold = {}
    for line in open(os.path.join(GOLDEN, "stencil_order.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, i, x, y, z = line.split()
        gold.setdefault(W.STENCILS[name], []).append((int(x), int(y), int(z)))
    for st in STENCILS:
        xi, *_ = oracle.tables(st)
        assert [tuple(v) for v in xi] == gold[st], st


def symmetry_generators(d):
    """Signed permutation matrices generating the square (2D) / cube (3D) symmetry group."""
    if d == 2:
        return [np.array([[0, 1, 0], [1, 0, 0], [0, 0, 1]]), np.diag([-1, 1, 1])]
    return [np.array([[0, 1, 0], [1, 0, 0], [0, 0, 1]]), np.array([[1, 0, 0], [0, 0, 1], [0, 1, 0]]),
            np.diag([-1, 1, 1])]


@pytest.mark.parametrize("st", STENCILS)
@pytest.mark.parametrize("space", [W.POPULATION, W.RAW, W.CENTRAL, W.CUMULANT])
def test_collision_isotropy(st, space):
    """With one rate per polynomial GROUP (rate set P) the collision commutes with every
    lattice symmetry: the grouped basis (reading R2) spans invariant subspaces, as the
    separation of shear, bulk and higher-order modes requires."""
    xi, opp, w, M, Minv = oracle.tables(st)
    fa = random_cells(st, 12, amp=5e-2)
    rates = np.array([1.3]) if space == W.POPULATION else W.rate_set_p(st)
    for eq, zc in admissible(space):
        fin = fa - w if zc else fa
        out = oracle.collide(st, space, eq, zc, rates, fin)
        for P in symmetry_generators(W.DIM_OF[st]):
            img = xi @ P.T
            perm = [int(np.flatnonzero((xi == img[i]).all(1))[0]) for i in range(len(w))]  # xi_perm[i] = P xi_i
            rot_in = np.empty_like(fin)
            rot_in[:, perm] = fin
            rot_out = oracle.collide(st, space, eq, zc, rates, rot_in)
            np.testing.assert_allclose(rot_out[:, perm], out, atol=2e-16, err_msg=f"{P}")


@pytest.mark.parametrize("st", STENCILS)
def test_moment_matrix_invertible(st):
    """M is invertible for the basis: M M^{-1} = I."""
    xi, opp, w, M, Minv = oracle.tables(st)
    q = W.Q_OF[st]
    assert np.linalg.matrix_rank(M) == q
    assert np.abs(M @ Minv - np.eye(q)).max() < 1e-14
    # row of p = 1 on w gives 1; p = x^2 gives cs^2
    assert (M[0] @ w) == pytest.approx(1.0, abs=1e-15)
    xx = (xi[:, 0] ** 2) @ w
    assert xx == pytest.approx(1 / 3, abs=1e-15)


# --------------------------------------------------- central moments / K ---
def raw_monomials(stencil, f):
    """m_abc = sum_i f_i xi_x^a xi_y^b xi_z^c (eq:DiscreteRawMomentsDef), all 27."""
    xi, *_ = oracle.tables(stencil)
    out = np.zeros((f.shape[0], 27))
    for k in range(27):
        e = (k % 3, (k // 3) % 3, k // 9)
        out[:, k] = f @ (xi[:, 0] ** e[0] * xi[:, 1] ** e[1] * xi[:, 2] ** e[2])
    return out


@pytest.mark.parametrize("st", STENCILS)
def test_central_moments_binomial(st):
    """kappa_abc = sum_{a'b'c'} C(a,a')C(b,b')C(c,c') (-u)^... m_a'b'c'
    (eq:RawToCentralMomentsBinomial); kappa_200 = m_200 - 2u m_100
    + u^2 m_000; at u = 0 central = raw (K(0) = M)."""
    f = random_cells(st, 20)
    k27, C27, rho, u = oracle.central_and_cumulants(st, f)
    m = raw_monomials(st, f)
    for k in range(27):
        e = (k % 3, (k // 3) % 3, k // 9)
        s = np.zeros(f.shape[0])
        for a in range(e[0] + 1):
            for b in range(e[1] + 1):
                for c in range(e[2] + 1):
                    coef = math.comb(e[0], a) * math.comb(e[1], b) * math.comb(e[2], c)
                    s += (coef * (-u[:, 0]) ** (e[0] - a) * (-u[:, 1]) ** (e[1] - b) * (-u[:, 2]) ** (e[2] - c)
                          * m[:, a + 3 * b + 9 * c])
        np.testing.assert_allclose(k27[:, k], s, atol=1e-15, rtol=1e-13)
    np.testing.assert_allclose(k27[:, 2], m[:, 2] - 2 * u[:, 0] * m[:, 1] + u[:, 0] ** 2 * m[:, 0], atol=1e-15)
    # kappa_000 = rho and kappa_100 = 0 (F = 0)
    np.testing.assert_allclose(k27[:, 0], rho, rtol=1e-15)
    assert np.abs(k27[:, [1, 3, 9]]).max() < 1e-16
    # u = 0: a distribution with zero momentum has central == raw moments
    xi, opp, w, M, Minv = oracle.tables(st)
    g = f.copy()
    g[:, :] = g[:, :] + g[:, opp]  # symmetric => zero momentum
    k0, _, _, u0 = oracle.central_and_cumulants(st, g)
    assert np.abs(u0).max() < 1e-16
    np.testing.assert_allclose(k0, raw_monomials(st, g), atol=1e-15)


# --------------------------------------------------------------- cumulants ---
def set_partitions(items):
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for part in set_partitions(rest):
        for k in range(len(part)):
            yield part[:k] + [[first] + part[k]] + part[k + 1:]
        yield [[first]] + part


def cumulant_by_partitions(stencil, f, e):
    """Classical moment-cumulant formula (Leonov-Shiryaev): the joint cumulant of
    the multiset of axes {x^a y^b z^c} of the normalised distribution f/rho is
    sum over set partitions pi of (-1)^{|pi|-1} (|pi|-1)! prod_B mu_B, mu = raw moments.
    Independent of the oracle's generating-function series."""
    xi, *_ = oracle.tables(stencil)
    rho = f.sum(1)
    labels = [0] * e[0] + [1] * e[1] + [2] * e[2]
    total = np.zeros(f.shape[0])
    for part in set_partitions(list(range(len(labels)))):
        k = len(part)
        term = (-1) ** (k - 1) * math.factorial(k - 1) * np.ones(f.shape[0])
        for B in part:
            v = np.ones(xi.shape[0])
            for idx in B:
                v = v * xi[:, labels[idx]]
            term = term * (f @ v) / rho
        total += term
    return rho * total  # rescaled C = rho c


@pytest.mark.parametrize("st", STENCILS)
def test_cumulants_partition_formula(st):
    """Every cumulant of order >= 2 equals the partition formula on raw moments."""
    f = random_cells(st, 12, amp=5e-2)
    k27, C27, rho, u = oracle.central_and_cumulants(st, f)
    for k in range(27):
        e = (k % 3, (k // 3) % 3, k // 9)
        if sum(e) < 2:
            continue
        if W.DIM_OF[st] == 2 and e[2] > 0:
            continue
        ref = cumulant_by_partitions(st, f, e)
        np.testing.assert_allclose(C27[:, k], ref, atol=2e-15, rtol=1e-12, err_msg=str(e))


@pytest.mark.parametrize("st", [W.D2Q9, W.D3Q27])
def test_cumulants_of_product_distribution(st):
    """Independent axes => every mixed cumulant vanishes; C_200 = rho Var_x
    (mutual statistical independence)."""
    rng = np.random.default_rng(11)
    xi, *_ = oracle.tables(st)
    n = 8
    d = W.DIM_OF[st]
    f = np.ones((n, xi.shape[0])) * rng.uniform(0.9, 1.1, (n, 1))
    var = np.zeros((n, 3))
    for a in range(d):
        p = rng.uniform(0.2, 1.0, (n, 3))
        p /= p.sum(1, keepdims=True)
        f *= p[np.arange(n)[:, None], xi[None, :, a] + 1]
        mean = p[:, 2] - p[:, 0]
        var[:, a] = p[:, 2] + p[:, 0] - mean ** 2
    k27, C27, rho, u = oracle.central_and_cumulants(st, f)
    for k in range(27):
        e = (k % 3, (k // 3) % 3, k // 9)
        if sum(e) < 2:
            continue
        nz = sum(1 for v in e if v > 0)
        if nz >= 2:
            assert np.abs(C27[:, k]).max() < 1e-16, e
    for a, k in enumerate([2, 6, 18][:d]):
        np.testing.assert_allclose(C27[:, k], rho * var[:, a], rtol=1e-14)


@pytest.mark.parametrize("st", STENCILS)
def test_cumulant_series_roundtrip(st):
    """K = exp(C - Xi.u) inverts C = Xi.u + log K (eq:CumulantAndCentralMomentGenFuncs)."""
    f = random_cells(st, 6, amp=5e-2)
    k27, C27, rho, u = oracle.central_and_cumulants(st, f)
    for c in range(f.shape[0]):
        back = oracle.cumulant_roundtrip(k27[c], rho[c])
        np.testing.assert_allclose(back, k27[c], atol=1e-16, rtol=1e-14)


# ------------------------------------------------------------- collision ---
@pytest.mark.parametrize("st", STENCILS)
@pytest.mark.parametrize("space", [W.POPULATION, W.RAW, W.CENTRAL, W.CUMULANT])
def test_collision_invariants(st, space):
    """Per cell: mass and momentum conserved; equilibrium is a fixed point;
    rates 0 => identity; rates 1 => f_eq."""
    xi, opp, w, M, Minv = oracle.tables(st)
    fa = random_cells(st, 30)
    rho = fa.sum(1)
    u = (fa @ xi) / rho[:, None]
    for eq, zc in admissible(space):
        rates = rates_for(st, space)
        fin = fa - w if zc else fa
        fo = oracle.collide(st, space, eq, zc, rates, fin)
        fo_abs = fo + w if zc else fo
        np.testing.assert_allclose(fo_abs.sum(1), rho, rtol=0, atol=1e-15)
        np.testing.assert_allclose(fo_abs @ xi, fa @ xi, rtol=0, atol=1e-16)
        feq = oracle.equilibrium(st, space, eq, zc, rho, u)
        np.testing.assert_allclose(oracle.collide(st, space, eq, zc, rates, feq), feq, atol=1e-16)
        r0 = oracle.collide(st, space, eq, zc, rates_for(st, space, 0.0), fin)
        np.testing.assert_allclose(r0, fin, atol=1e-16)
        r1 = oracle.collide(st, space, eq, zc, rates_for(st, space, 1.0), fin)
        np.testing.assert_allclose(r1, feq, atol=1e-16)


@pytest.mark.parametrize("st", STENCILS)
@pytest.mark.parametrize("space", LINEAR_SPACES)
def test_background_invariance(st, space):
    """delta f = 0 stays 0 in the deviation-only regime.  For
    CENTRAL the oracle forms dq_eq = q_eq - T(f0) literally with the
    numerically inverted f0, so it is zero only to long-double rounding."""
    q = W.Q_OF[st]
    fo = oracle.collide(st, space, W.EQ_DELTA, 1, rates_for(st, space), np.zeros((3, q)))
    if space == W.CENTRAL:
        assert np.abs(fo).max() < 1e-18
    else:
        assert (fo == 0).all()


@pytest.mark.parametrize("st", [W.D2Q9, W.D3Q27])
def test_bgk_equivalence(st):
    """All rates equal: RAW reduces to BGK with the textbook Hermite f_eq; CENTRAL
    and CUMULANT (omega = 1) to BGK with the Gaussian product f_eq."""
    xi, opp, w, M, Minv = oracle.tables(st)
    fa = random_cells(st, 25)
    rho = fa.sum(1)
    u = (fa @ xi) / rho[:, None]
    om = 1.37
    ref_raw = fa + om * (textbook_feq(st, rho, u) - fa)
    ref_cm = fa + om * (product_feq(st, rho, u) - fa)
    for eq, zc in ALL_REGIMES:
        fin = fa - w if zc else fa
        back = (lambda x: x + w) if zc else (lambda x: x)
        np.testing.assert_allclose(back(oracle.collide(st, W.RAW, eq, zc, rates_for(st, W.RAW, om), fin)),
                                   ref_raw, atol=1e-16)
        np.testing.assert_allclose(back(oracle.collide(st, W.POPULATION, eq, zc, [om], fin)), ref_raw, atol=1e-16)
        np.testing.assert_allclose(back(oracle.collide(st, W.CENTRAL, eq, zc, rates_for(st, W.CENTRAL, om), fin)),
                                   ref_cm, atol=1e-16)
    for zc in (0, 1):
        fin = fa - w if zc else fa
        out = oracle.collide(st, W.CUMULANT, W.EQ_ABSOLUTE, zc, rates_for(st, W.CUMULANT, 1.0), fin)
        np.testing.assert_allclose(out + (w if zc else 0), product_feq(st, rho, u), atol=1e-16)
        # and K is NOT BGK at omega != 1 (nonlinear transform)
        out = oracle.collide(st, W.CUMULANT, W.EQ_ABSOLUTE, zc, rates_for(st, W.CUMULANT, om), fin)
        assert np.abs(out + (w if zc else 0) - ref_cm).max() > 1e-9


def test_d3q19_equilibrium_moments():
    """On D3Q19 the equilibrium is M^{-1} m_eq with m_eq the Maxwellian moments
    truncated at O(u^2) (reading R4); hand-derived values."""
    st = W.D3Q19
    rng = np.random.default_rng(5)
    n = 10
    rho = rng.uniform(0.95, 1.05, n)
    u = rng.uniform(-0.1, 0.1, (n, 3))
    f = oracle.equilibrium(st, W.RAW, W.EQ_ABSOLUTE, 0, rho, u)
    m = raw_monomials(st, f)
    ux, uy, uz = u.T
    idx = lambda a, b, c: a + 3 * b + 9 * c
    np.testing.assert_allclose(m[:, idx(0, 0, 0)], rho, rtol=1e-15)
    np.testing.assert_allclose(m[:, idx(1, 0, 0)], rho * ux, atol=1e-16)
    np.testing.assert_allclose(m[:, idx(1, 1, 0)], rho * ux * uy, atol=1e-16)
    np.testing.assert_allclose(m[:, idx(2, 0, 0)], rho * (1 / 3 + ux ** 2), atol=1e-16)
    np.testing.assert_allclose(m[:, idx(2, 1, 0)], rho * uy / 3, atol=1e-16)
    np.testing.assert_allclose(m[:, idx(1, 0, 2)], rho * ux / 3, atol=1e-16)
    np.testing.assert_allclose(m[:, idx(2, 2, 0)], rho * (1 / 9 + (ux ** 2 + uy ** 2) / 3), atol=1e-16)
    np.testing.assert_allclose(m[:, idx(0, 2, 2)], rho * (1 / 9 + (uy ** 2 + uz ** 2) / 3), atol=1e-16)
    # ... which differs from the textbook D3Q19 polynomial by -rho uz^2 / 6 in m_220
    mt = raw_monomials(st, textbook_feq(st, rho, u))
    np.testing.assert_allclose(mt[:, idx(2, 2, 0)] - m[:, idx(2, 2, 0)], -rho * uz ** 2 / 6, atol=1e-16)


@pytest.mark.parametrize("st", STENCILS)
@pytest.mark.parametrize("space", [W.POPULATION, W.RAW, W.CENTRAL, W.CUMULANT])
def test_regime_equivalence(st, space):
    """absolute == zc + delta eq == zc + absolute eq under delta f = f - f0
    (SPEC.md:508)."""
    xi, opp, w, M, Minv = oracle.tables(st)
    fa = random_cells(st, 20)
    rates = rates_for(st, space)
    outs = []
    for eq, zc in admissible(space):
        fin = fa - w if zc else fa
        o = oracle.collide(st, space, eq, zc, rates, fin)
        outs.append(o + w if zc else o)
    for o in outs[1:]:
        np.testing.assert_allclose(o, outs[0], atol=1.2e-16, rtol=0)  # ~1 ulp of the absolute populations (double output of + w)


# ------------------------------------------------------ streaming / bc ---
@pytest.mark.parametrize("st", STENCILS)
def test_pull_moves_population_by_xi(st):
    """eq:LbStreaming: with an identity collision (rate 0) a single
    population travels one node along xi_i per step, wrapping periodically."""
    xi, opp, w, M, Minv = oracle.tables(st)
    q = W.Q_OF[st]
    nx, ny, nz = (5, 4, 1) if st == W.D2Q9 else (5, 4, 6)
    sim = oracle.Sim(st, W.POPULATION, W.EQ_DELTA, 1, [0.0], (nx, ny, nz))
    for i in range(q):
        f = np.zeros((q, nz, ny, nx))
        x0, y0, z0 = 4, 0, nz - 1  # at the high/low edges to exercise the wrap
        f[i, z0, y0, x0] = 1.0
        sim.set(f)
        sim.step(2)
        g = sim.get()
        x1, y1, z1 = (x0 + 2 * xi[i, 0]) % nx, (y0 + 2 * xi[i, 1]) % ny, (z0 + 2 * xi[i, 2]) % nz
        assert g[i, z1, y1, x1] == 1.0
        assert np.count_nonzero(g) == 1


def test_bounce_back_reverses_population():
    """Half-way bounce-back (reading R18): a population leaving through a no-slip
    face returns to its node in the opposite slot one step later."""
    st = W.D3Q19
    xi, opp, w, M, Minv = oracle.tables(st)
    q = 19
    nx, ny, nz = 4, 5, 6
    bc = [[W.PERIODIC, W.PERIODIC], [W.PERIODIC, W.PERIODIC], [W.NOSLIP, W.NOSLIP]]
    sim = oracle.Sim(st, W.POPULATION, W.EQ_DELTA, 1, [0.0], (nx, ny, nz), bc=bc)
    for i in range(q):
        if xi[i, 2] == 0:
            continue
        f = np.zeros((q, nz, ny, nx))
        z0 = nz - 1 if xi[i, 2] > 0 else 0
        f[i, z0, 2, 1] = 1.0
        sim.set(f)
        sim.step(1)
        g = sim.get()
        assert g[opp[i], z0, 2, 1] == 1.0 and np.count_nonzero(g) == 1


def test_mass_conserved_with_walls():
    st = W.D3Q27
    xi, opp, w, M, Minv = oracle.tables(st)
    nx, ny, nz = 6, 5, 7
    bc = [[W.NOSLIP, W.NOSLIP], [W.PERIODIC, W.PERIODIC], [W.NOSLIP, W.NOSLIP]]
    sim = oracle.Sim(st, W.CUMULANT, W.EQ_ABSOLUTE, 1, W.rate_set_p(st), (nx, ny, nz), bc=bc)
    rng = np.random.default_rng(2)
    f = 1e-2 * w[:, None, None, None] * rng.uniform(-1, 1, (27, nz, ny, nx))
    sim.set(f)
    m0 = f.sum()
    sim.step(5)
    assert abs(sim.get().sum() - m0) < 1e-14


# ----------------------------------------------------------------- physics ---
def run_tgv(st, space, eq, zc, nu, u0, L, steps, prec=oracle.LONG_DOUBLE):
    xi, opp, w, M, Minv = oracle.tables(st)
    om = W.omega_from_nu(nu)
    rates = [om] if space == W.POPULATION else W.regularized_rates(st, om)
    rho, u = W.tgv_fields(L, L, 1, u0)
    feq = oracle.equilibrium(st, space, eq, zc, rho.reshape(-1), u.reshape(3, -1).T)
    sim = oracle.Sim(st, space, eq, zc, rates, (L, L, 1), prec=prec)
    sim.set(np.ascontiguousarray(feq.T.reshape(W.Q_OF[st], 1, L, L)))

    def energy():
        r, uu = sim.macroscopic()
        return 0.5 * (r * (uu ** 2).sum(0)).sum()

    e0 = energy()
    sim.step(steps)
    return energy() / e0


@pytest.mark.parametrize("space,eq,zc,nu", [
    (W.POPULATION, W.EQ_DELTA, 1, 1 / 6),
    (W.POPULATION, W.EQ_DELTA, 1, 0.02),
    (W.RAW, W.EQ_DELTA, 1, 0.05),
    (W.CENTRAL, W.EQ_ABSOLUTE, 1, 0.05),
    (W.CUMULANT, W.EQ_ABSOLUTE, 1, 0.05),
    (W.CENTRAL, W.EQ_DISCRETE, 1, 0.05),
    (W.CUMULANT, W.EQ_DISCRETE, 1, 0.05),
    (W.RAW, W.EQ_DISCRETE_DELTA, 1, 0.05),
])
def test_tgv_energy_decay(space, eq, zc, nu):
    """E/E0 = exp(-4 nu kappa^2 t) (eq:TGA_kin_energy) within 1 %
    at u0 = 0.05, L = 48, 300 steps; the shear group of reading R3 sets nu."""
    L, steps = 48, 300
    ratio = run_tgv(W.D2Q9, space, eq, zc, nu, 0.05, L, steps)
    ref = W.tgv_energy_ratio(nu, L, steps)
    assert abs(ratio / ref - 1) < 1e-2, (ratio, ref)


@pytest.mark.parametrize("space,eq,zc", [
    (W.POPULATION, W.EQ_DELTA, 1), (W.RAW, W.EQ_DELTA, 1), (W.CENTRAL, W.EQ_ABSOLUTE, 1),
    (W.CUMULANT, W.EQ_ABSOLUTE, 1),
])
def test_tgv_second_order_convergence(space, eq, zc):
    """The deviation of E/E0 from exp(-4 nu kappa^2 t) (eq:TGA_kin_energy) converges at second
    order under diffusive scaling (L = 16, 32, 64; u0 = 0.05 * 32 / L; t to E/E0 ~ 1/2): the
    error ratio between successive lattices is 4 (LBM is second-order accurate in space; the
    Mach-number error u0^2 shrinks at the same rate)."""
    nu = 0.05
    errs = []
    for L in (16, 32, 64):
        k = 2 * math.pi / L
        steps = int(round(math.log(2) / (4 * nu * k * k)))
        ratio = run_tgv(W.D2Q9, space, eq, zc, nu, 0.05 * 32 / L, L, steps, prec=oracle.DOUBLE)
        errs.append(abs(ratio / W.tgv_energy_ratio(nu, L, steps) - 1))
    for a, b in zip(errs, errs[1:]):
        assert 3.6 < a / b < 4.4, errs


FORCE = np.array([2e-4, -1e-4, 3e-4])


@pytest.mark.parametrize("model", [oracle.GUO, oracle.HE])
@pytest.mark.parametrize("st", STENCILS)
@pytest.mark.parametrize("space", [W.POPULATION, W.RAW, W.CENTRAL, W.CUMULANT])
def test_force_momentum_and_paper_example(st, space, model):
    """Body force (readings R23, R26, R27): per cell the mass is unchanged and the momentum gains
    F; written as the paper's worked example: with u = (j + F/2)/rho the
    post-collision first-order raw moment is m*_{10|0} = rho u_x + F_x / 2."""
    xi, opp, w, M, Minv = oracle.tables(st)
    F = FORCE.copy()
    if W.DIM_OF[st] == 2:
        F[2] = 0
    fa = random_cells(st, 20)
    rho = fa.sum(1)
    u = (fa @ xi + F / 2) / rho[:, None]  # pre-collision velocity with the half-force shift
    for eq, zc in admissible(space):
        fin = fa - w if zc else fa
        fo = oracle.collide(st, space, eq, zc, rates_for(st, space), fin, force=F, force_model=model)
        fo_abs = fo + w if zc else fo
        np.testing.assert_allclose(fo_abs.sum(1), rho, atol=1e-15)
        np.testing.assert_allclose(fo_abs @ xi, rho[:, None] * u + F / 2, atol=1e-16)


def cells_with_velocity(st, n, u_dir, speed, F, seed=11, amp=2e-2):
    """Absolute populations with the SHIFTED velocity (j + F/2)/rho = speed * u_dir exactly:
    random non-equilibrium noise, then the momentum corrected along a zero-mass direction."""
    xi, opp, w, M, Minv = oracle.tables(st)
    rng = np.random.default_rng(seed)
    rho = 1.0 + rng.uniform(-0.03, 0.03, n)
    u = np.tile(speed * np.asarray(u_dir, float), (n, 1))
    f = textbook_feq(st, rho, u) + amp * w * rng.uniform(-1, 1, (n, len(w)))
    d = W.DIM_OF[st]
    for _ in range(2):  # set sum f = rho and sum f xi = rho u - F/2 with w-weighted corrections
        f += w * (rho - f.sum(1))[:, None]
        dj = rho[:, None] * u - F / 2 - f @ xi
        f += 3.0 * w * (dj[:, :d] @ xi[:, :d].T)
    return f


@pytest.mark.parametrize("st,space", [(W.D2Q9, W.POPULATION), (W.D3Q19, W.RAW), (W.D3Q27, W.CENTRAL),
                                      (W.D2Q9, W.CENTRAL)])
def test_he_force_equals_guo_at_rest(st, space):
    """Reading R27: at u = 0 He's term f_eq (xi - u).F/(rho c_s^2) is rho w_i 3 xi.F / rho, which
    is Guo's w_i [3 xi.F + 9 (xi.u)(xi.F) - 3 u.F] at u = 0 — the two forced collisions agree."""
    xi, opp, w, M, Minv = oracle.tables(st)
    F = FORCE.copy()
    if W.DIM_OF[st] == 2:
        F[2] = 0
    fa = cells_with_velocity(st, 10, [1, 0, 0], 0.0, F)
    np.testing.assert_allclose((fa @ xi + F / 2), 0, atol=1e-15)
    rates = rates_for(st, space)
    for eq, zc in admissible(space):
        fin = fa - w if zc else fa
        g = oracle.collide(st, space, eq, zc, rates, fin, force=F, force_model=oracle.GUO)
        h = oracle.collide(st, space, eq, zc, rates, fin, force=F, force_model=oracle.HE)
        np.testing.assert_allclose(h, g, atol=2e-17)


@pytest.mark.parametrize("st,space", [(W.D2Q9, W.POPULATION), (W.D3Q27, W.RAW), (W.D3Q27, W.CENTRAL)])
def test_he_minus_guo_is_second_order_in_u(st, space):
    """Reading R27: He's and Guo's terms agree to first order in u (both carry the (xi.u)(xi.F)
    term of the second-order expansion), so the forced collisions differ by O(u^2 F): halving u
    quarters the difference.  A wrong sign or a missing (xi - u) shift breaks the ratio."""
    F = FORCE.copy()
    if W.DIM_OF[st] == 2:
        F[2] = 0
    xi, opp, w, M, Minv = oracle.tables(st)
    rates = rates_for(st, space)
    diffs = []
    for speed in (0.04, 0.02, 0.01):
        fa = cells_with_velocity(st, 6, [0.6, -0.8, 0.0] if W.DIM_OF[st] == 2 else [0.48, -0.64, 0.6], speed, F)
        g = oracle.collide(st, space, W.EQ_ABSOLUTE, 0, rates, fa, force=F, force_model=oracle.GUO)
        h = oracle.collide(st, space, W.EQ_ABSOLUTE, 0, rates, fa, force=F, force_model=oracle.HE)
        diffs.append(np.abs(h - g).max())
    assert diffs[0] > 1e-3 * 0.04 ** 2 * np.abs(F).max()  # the models are not identical
    for a, b in zip(diffs, diffs[1:]):
        assert 3.6 < a / b < 4.4, diffs


def test_force_cumulant_models_coincide():
    """Reading R26/R27: for the cumulant methods both models give the first-order source F."""
    st = W.D3Q27
    xi, opp, w, M, Minv = oracle.tables(st)
    fa = random_cells(st, 6)
    rates = rates_for(st, W.CUMULANT)
    g = oracle.collide(st, W.CUMULANT, W.EQ_ABSOLUTE, 1, rates, fa - w, force=FORCE, force_model=oracle.GUO)
    h = oracle.collide(st, W.CUMULANT, W.EQ_ABSOLUTE, 1, rates, fa - w, force=FORCE, force_model=oracle.HE)
    np.testing.assert_array_equal(g, h)


def test_force_shallow_water_unsupported():
    """No force model for the shallow-water methods (reading R23)."""
    xi, opp, w, M, Minv = oracle.tables(W.D2Q9)
    f = np.tile(2.0 * w, (3, 1))
    for space in (W.CENTRAL, W.CUMULANT):
        with pytest.raises(RuntimeError):
            oracle.collide(W.D2Q9, space, W.EQ_SWE, 0, W.rate_set_p(W.D2Q9), f, g=0.0613125,
                           force=[1e-4, 0, 0])


@pytest.mark.parametrize("st", [W.D2Q9, W.D3Q27])
def test_cumulant_force_is_first_order_only(st):
    """Reading R26: the cumulant source q^F is F on the first-order cumulants and zero on every
    cumulant of order >= 2.  Cumulants of order >= 2 do not depend on the frame (PAPER.md:411,
    eq:CumulantAndCentralMomentGenFuncs), so the forced and the unforced collision of the same
    cell leave IDENTICAL cumulants of order >= 2 (computed from the outputs by the pinned
    generating-function transform) and differ in momentum by exactly F.  Full stencils only:
    there the populations determine all 3^d monomial cumulants."""
    xi, opp, w, M, Minv = oracle.tables(st)
    F = FORCE.copy()
    if W.DIM_OF[st] == 2:
        F[2] = 0
    fa = random_cells(st, 12)
    rates = W.rates_random(st, seed=5)
    plain = oracle.collide(st, W.CUMULANT, W.EQ_ABSOLUTE, 0, rates, fa)
    forced = oracle.collide(st, W.CUMULANT, W.EQ_ABSOLUTE, 0, rates, fa, force=F)
    _, c_plain, _, _ = oracle.central_and_cumulants(st, plain)
    _, c_forced, _, _ = oracle.central_and_cumulants(st, forced)
    order = np.array([k % 3 + (k // 3) % 3 + k // 9 for k in range(27)])
    hi = order >= 2
    np.testing.assert_allclose(c_forced[:, hi], c_plain[:, hi], atol=1e-15)
    assert np.abs(c_forced[:, hi] - c_plain[:, hi]).max() < 1e-3 * np.abs(F).max()
    np.testing.assert_allclose(forced @ xi - plain @ xi, np.tile(F, (len(fa), 1)), atol=1e-16)
    np.testing.assert_allclose(forced.sum(1), plain.sum(1), atol=1e-15)


@pytest.mark.parametrize("model", [oracle.GUO, oracle.HE])
@pytest.mark.parametrize("st", STENCILS)
@pytest.mark.parametrize("space", [W.POPULATION, W.RAW, W.CENTRAL, W.CUMULANT])
def test_force_isotropy(st, space, model):
    """Rotating the cell and the force together commutes with the forced collision."""
    xi, opp, w, M, Minv = oracle.tables(st)
    F = FORCE.copy()
    if W.DIM_OF[st] == 2:
        F[2] = 0
    fa = random_cells(st, 8)
    rates = np.array([1.3]) if space == W.POPULATION else W.rate_set_p(st)
    eq = W.EQ_ABSOLUTE if space == W.CUMULANT else W.EQ_DELTA
    out = oracle.collide(st, space, eq, 1, rates, fa - w, force=F, force_model=model)
    for P in symmetry_generators(W.DIM_OF[st]):
        img = xi @ P.T
        perm = [int(np.flatnonzero((xi == img[i]).all(1))[0]) for i in range(len(w))]
        rot_in = np.empty_like(fa)
        rot_in[:, perm] = fa - w
        rot_out = oracle.collide(st, space, eq, 1, rates, rot_in, force=P @ F, force_model=model)
        np.testing.assert_allclose(rot_out[:, perm], out, atol=2e-16)


@pytest.mark.parametrize("space,nu,model", [(W.POPULATION, 1 / 6, oracle.GUO), (W.RAW, 0.1, oracle.GUO),
                                            (W.CENTRAL, 0.05, oracle.GUO), (W.CUMULANT, 0.08, oracle.GUO),
                                            (W.POPULATION, 0.1, oracle.HE), (W.CENTRAL, 0.05, oracle.HE)])
def test_poiseuille_flow(space, nu, model):
    """Force-driven channel between half-way bounce-back walls (readings R18, R23): the steady
    profile is u_x(y) = F / (2 nu) (y + 1/2)(H - 1/2 - y) (walls half a node outside)."""
    st, nx, ny, Fx = W.D2Q9, 4, 24, 1e-6
    om = W.omega_from_nu(nu)
    rates = [om] if space == W.POPULATION else W.regularized_rates(st, om)
    bc = [[W.PERIODIC, W.PERIODIC], [W.NOSLIP, W.NOSLIP], [W.PERIODIC, W.PERIODIC]]
    eq = W.EQ_ABSOLUTE if space == W.CUMULANT else W.EQ_DELTA
    sim = oracle.Sim(st, space, eq, 1, rates, (nx, ny, 1), bc=bc)
    sim.set(np.zeros((9, 1, ny, nx)))
    sim.set_force([Fx, 0, 0], force_model=model)
    sim.step(int(8 * ny * ny / nu))
    r, u = sim.macroscopic()
    y = np.arange(ny)
    ref = Fx / (2 * nu) * (y + 0.5) * (ny - 0.5 - y)
    assert np.abs(u[0, 0, :, 0] - ref).max() < 1e-2 * ref.max()
    assert np.abs(u[1]).max() < 1e-12 * ref.max()


@pytest.mark.parametrize("st,space,tau,model", [
    (W.D2Q9, W.POPULATION, 1.0, oracle.GUO), (W.D2Q9, W.POPULATION, 0.65, oracle.HE),
    (W.D2Q9, W.POPULATION, 0.5 + np.sqrt(3 / 16), oracle.GUO), (W.D2Q9, W.RAW, 0.8, oracle.GUO),
    (W.D2Q9, W.CENTRAL, 1.1, oracle.GUO), (W.D2Q9, W.CUMULANT, 0.875, oracle.HE),
    (W.D3Q19, W.RAW, 0.875, oracle.GUO), (W.D3Q27, W.POPULATION, 0.65, oracle.GUO),
    (W.D3Q27, W.CUMULANT, 1.1, oracle.GUO)])
def test_poiseuille_bounce_back_closed_form(st, space, tau, model):
    """Half-way bounce-back (reading R18) pinned by a closed form of the LB literature rather
    than by the paper (which has no walls): for a force-driven channel the steady discrete
    solution is EXACTLY the parabola with the walls half a node outside plus a uniform slip,
        u_x(y) = F / (2 nu) [ (y + 1/2)(H - 1/2 - y) + (16 Lambda - 3) / 12 ],
    with Lambda = (tau_s - 1/2)(tau_odd - 1/2) the product of the even (shear) and odd
    relaxation times (BGK: tau_odd = tau_s; the R- methods: odd moments at rate 1, tau_odd = 1);
    bounce-back is exact at Lambda = 3/16 (Ginzburg & d'Humieres 2003).  A reversed or
    misplaced bounce, a wrong force sign or half-force velocity shift, or a wrong rate slot all
    change the slip or the curvature."""
    nx, ny, Fx = 2, 8, 1e-6
    nz = 1 if W.DIM_OF[st] == 2 else 2
    nu = (tau - 0.5) / 3
    rates = [1 / tau] if space == W.POPULATION else W.regularized_rates(st, 1 / tau)
    lam = (tau - 0.5) * ((tau - 0.5) if space == W.POPULATION else 0.5)
    bc = [[W.PERIODIC, W.PERIODIC], [W.NOSLIP, W.NOSLIP], [W.PERIODIC, W.PERIODIC]]
    eq = W.EQ_ABSOLUTE if space == W.CUMULANT else W.EQ_DELTA
    sim = oracle.Sim(st, space, eq, 1, rates, (nx, ny, nz), bc=bc)
    sim.set(np.zeros((W.Q_OF[st], nz, ny, nx)))
    sim.set_force([Fx, 0, 0], force_model=model)
    sim.step(30000)  # >= 25 diffusion times H^2 / nu: converged to ~1e-11
    _, u = sim.macroscopic()
    y = np.arange(ny)
    ref = Fx / (2 * nu) * ((y + 0.5) * (ny - 0.5 - y) + (16 * lam - 3) / 12)
    for z in range(nz):
        for x in range(nx):
            assert np.abs(u[0, z, :, x] - ref).max() < 1e-9 * ref.max()
    assert np.abs(u[1:]).max() < 1e-12 * ref.max()


def test_shear_wave_between_walls():
    """Bounce-back pin (reading R18): u_x(y) = u0 sin(pi (y+1/2)/ny) between no-slip
    walls decays as exp(-nu (pi/ny)^2 t)."""
    st = W.D2Q9
    nx, ny, steps, u0, nu = 4, 24, 200, 1e-3, 1 / 6
    y = np.arange(ny)
    ux = u0 * np.sin(np.pi * (y + 0.5) / ny)
    rho = np.ones((ny, nx)).reshape(-1)
    u = np.zeros((ny * nx, 3))
    u[:, 0] = np.repeat(ux, nx)
    feq = oracle.equilibrium(st, W.POPULATION, W.EQ_DELTA, 1, rho, u)
    bc = [[W.PERIODIC, W.PERIODIC], [W.NOSLIP, W.NOSLIP], [W.PERIODIC, W.PERIODIC]]
    sim = oracle.Sim(st, W.POPULATION, W.EQ_DELTA, 1, [W.omega_from_nu(nu)], (nx, ny, 1), bc=bc)
    sim.set(np.ascontiguousarray(feq.T.reshape(9, 1, ny, nx)))
    sim.step(steps)
    r, uu = sim.macroscopic()
    amp = (uu[0, 0, :, 0] * np.sin(np.pi * (y + 0.5) / ny)).sum() / (np.sin(np.pi * (y + 0.5) / ny) ** 2).sum()
    ref = u0 * math.exp(-nu * (math.pi / ny) ** 2 * steps)
    assert abs(amp / ref - 1) < 1e-2


@pytest.mark.parametrize("space", [W.CENTRAL, W.CUMULANT])
def test_swe_equilibrium_moments(space):
    """Corrected eq:DiscreteShallowWaterEquilibrium (reading R5) for the CM method and the
    Maxwellian with cs2 = g h / 2 for the cumulant method: sum f = h,
    sum f xi = h u, sum f xi_a xi_b = h u_a u_b + g h^2/2 delta_ab (Zhou 2002)."""
    st = W.D2Q9
    xi, *_ = oracle.tables(st)
    rng = np.random.default_rng(9)
    n, g = 10, 0.0613125
    h = rng.uniform(1.0, 6.0, n)
    u = np.zeros((n, 3))
    u[:, :2] = rng.uniform(-0.1, 0.1, (n, 2))
    f = oracle.equilibrium(st, space, W.EQ_SWE, 0, h, u, g=g)
    if space == W.CUMULANT:
        # product (Gaussian) form: variance cs2 = g h / 2 per axis, no mixed cumulants
        k27, C27, rho, uu = oracle.central_and_cumulants(st, f)
        np.testing.assert_allclose(C27[:, 2], h * g * h / 2, rtol=1e-14)
        np.testing.assert_allclose(C27[:, 6], h * g * h / 2, rtol=1e-14)
        assert np.abs(C27[:, [4, 5, 7, 8]]).max() < 1e-15
    np.testing.assert_allclose(f.sum(1), h, rtol=1e-15)
    np.testing.assert_allclose(f @ xi[:, :2], h[:, None] * u[:, :2], atol=1e-15)
    for a in range(2):
        for b in range(2):
            P = f @ (xi[:, a] * xi[:, b])
            ref = h * u[:, a] * u[:, b] + (g * h * h / 2 if a == b else 0)
            np.testing.assert_allclose(P, ref, atol=1e-14)


@pytest.mark.parametrize("space", [W.CENTRAL, W.CUMULANT])
def test_swe_collision_conserves(space):
    """Both shallow-water methods conserve h and h u per cell, keep their equilibrium
    fixed, and reach it with every rate one."""
    st = W.D2Q9
    xi, *_ = oracle.tables(st)
    rng = np.random.default_rng(4)
    n, g = 10, 0.0613125
    h = rng.uniform(1.0, 6.0, n)
    u = np.zeros((n, 3))
    u[:, :2] = rng.uniform(-0.05, 0.05, (n, 2))
    feq = oracle.equilibrium(st, space, W.EQ_SWE, 0, h, u, g=g)
    f = feq * (1 + 0.02 * rng.uniform(-1, 1, feq.shape))
    rates = W.regularized_rates(st, 0.695652)
    fo = oracle.collide(st, space, W.EQ_SWE, 0, rates, f, g=g)
    np.testing.assert_allclose(fo.sum(1), f.sum(1), rtol=1e-15)
    np.testing.assert_allclose(fo @ xi, f @ xi, atol=1e-15)
    np.testing.assert_allclose(oracle.collide(st, space, W.EQ_SWE, 0, rates, feq, g=g), feq, atol=1e-15)
    h2 = f.sum(1)
    u2 = np.zeros((n, 3))
    u2[:, :2] = (f @ xi[:, :2]) / h2[:, None]
    np.testing.assert_allclose(oracle.collide(st, space, W.EQ_SWE, 0, np.ones(9), f, g=g),
                               oracle.equilibrium(st, space, W.EQ_SWE, 0, h2, u2, g=g), atol=1e-15)


@pytest.mark.parametrize("space", [W.CENTRAL, W.CUMULANT])
def test_swe_zero_centered_storage(space):
    """Zero-centered shallow water (reading R33): the background is the
    method's rest state f0 = f_eq(h0 = 1, u = 0), typed here from its definitions — Zhou's
    f0 = (1 - 5g/6; g/6 on the axes; g/24 on the diagonals) and, for the cumulant method, the
    product of the per-axis Gaussian moment conditions at cs2 = g/2 (phi(0) = 1 - cs2,
    phi(+-1) = cs2 / 2); the rest state df = 0 is a fixed point; and the zero-centered update
    equals the absolute one under df = f - f0 to one ulp."""
    st = W.D2Q9
    xi, *_ = oracle.tables(st)
    g = 0.0613125
    f0 = oracle.equilibrium(st, space, W.EQ_SWE, 0, np.ones(1), np.zeros((1, 3)), g=g)[0]
    if space == W.CENTRAL:
        l1 = np.abs(xi[:, :2]).sum(1)
        typed = np.where(l1 == 0, 1 - 5 * g / 6, np.where(l1 == 1, g / 6, g / 24))
    else:
        cs2 = g / 2
        phi = lambda x: np.where(x == 0, 1 - cs2, cs2 / 2)
        typed = phi(xi[:, 0]) * phi(xi[:, 1])
    np.testing.assert_allclose(f0, typed, rtol=2e-16, atol=1e-17)
    # zero-centered rest state: equilibrium 0, collision fixed point
    z = oracle.equilibrium(st, space, W.EQ_SWE, 1, np.ones(1), np.zeros((1, 3)), g=g)
    assert np.abs(z).max() < 1e-17
    rates = W.rates_random(st)
    assert np.abs(oracle.collide(st, space, W.EQ_SWE, 1, rates, np.zeros((3, 9)), g=g)).max() < 1e-17
    # regime equivalence on perturbed states
    rng = np.random.default_rng(8)
    n = 16
    h = rng.uniform(1.0, 6.0, n)
    u = np.zeros((n, 3))
    u[:, :2] = rng.uniform(-0.05, 0.05, (n, 2))
    fa = oracle.equilibrium(st, space, W.EQ_SWE, 0, h, u, g=g) * (1 + 0.02 * rng.uniform(-1, 1, (n, 9)))
    oa = oracle.collide(st, space, W.EQ_SWE, 0, rates, fa, g=g)
    oz = oracle.collide(st, space, W.EQ_SWE, 1, rates, fa - f0, g=g) + f0
    np.testing.assert_allclose(oz, oa, rtol=0, atol=1e-15)
    fz = oracle.equilibrium(st, space, W.EQ_SWE, 1, h, u, g=g)
    np.testing.assert_allclose(fz + f0, oracle.equilibrium(st, space, W.EQ_SWE, 0, h, u, g=g), atol=1e-15)


def paper_values():
    vals = {}
    for line in open(os.path.join(GOLDEN, "paper_values.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, v, tol, cite = line.split(None, 3)
        vals[k] = (float(v), float(tol))
    return vals


def test_paper_values():
    vals = paper_values()
    g, nu, om = W.swe_lattice_parameters()
    v, tol = vals["dam_break_omega_s"]
    assert abs(om - v) < tol
    v, tol = vals["tgv_omega_at_nu_1_6"]
    assert abs(W.omega_from_nu(1 / 6) - v) < tol
    v, tol = vals["tgv_rho_origin_u0_0.25"]
    rho, u = W.tgv_fields(8, 8, 1, 0.25)
    assert abs(rho[0, 0, 0] - v) < tol


# ----------------------------------------------------------- discrete equilibrium (reading R29)
DISC_REGIMES = [(W.EQ_DISCRETE, 0), (W.EQ_DISCRETE_DELTA, 1), (W.EQ_DISCRETE, 1)]


def _abs(f, w, eq, zc):
    return f + w if zc else f


@pytest.mark.parametrize("st", [W.D2Q9, W.D3Q27])
@pytest.mark.parametrize("space", [W.POPULATION, W.RAW])
def test_discrete_equals_continuous_for_full_stencils(st, space):
    """On D2Q9 and D3Q27 the truncated continuous Maxwellian's raw moments ARE those of the
    textbook discrete f_eq (reading R4), so the two equilibrium forms give the same SRT and
    raw-moment collision in every regime (q_eq = T(f_eq))."""
    xi, opp, w, M, Minv = oracle.tables(st)
    fa = random_cells(st, 10)
    rates = rates_for(st, space)
    for (deq, zc), (ceq, _) in zip(DISC_REGIMES, ALL_REGIMES):
        fin = fa - w if zc else fa
        d = oracle.collide(st, space, deq, zc, rates, fin)
        c = oracle.collide(st, space, ceq, zc, rates, fin)
        np.testing.assert_allclose(d, c, atol=2e-17)


def test_discrete_d3q19_differs_and_is_bgk():
    """D3Q19: the discrete f_eq differs from M^-1 m_eq of the truncated Maxwellian (by the
    -rho u_z^2/6 terms of reading R4), and SRT with it is BGK with the textbook polynomial."""
    st = W.D3Q19
    xi, opp, w, M, Minv = oracle.tables(st)
    fa = random_cells(st, 10)
    rho = fa.sum(1)
    u = (fa @ xi) / rho[:, None]
    om = 1.3
    d = oracle.collide(st, W.POPULATION, W.EQ_DISCRETE, 0, [om], fa)
    c = oracle.collide(st, W.POPULATION, W.EQ_ABSOLUTE, 0, [om], fa)
    np.testing.assert_allclose(d, fa + om * (textbook_feq(st, rho, u) - fa), atol=1e-16)
    assert np.abs(d - c).max() > 1e-7
    rates = rates_for(st, W.RAW)
    assert np.abs(oracle.collide(st, W.RAW, W.EQ_DISCRETE, 0, rates, fa)
                  - oracle.collide(st, W.RAW, W.EQ_ABSOLUTE, 0, rates, fa)).max() > 1e-7


@pytest.mark.parametrize("st", STENCILS)
def test_discrete_central_moments_at_equal_rates_is_bgk(st):
    """T = K(u) is linear: relaxing every central moment at the same rate towards K(u) f_eq is
    f* = f + omega (f_eq - f) with the textbook discrete f_eq, in every regime."""
    xi, opp, w, M, Minv = oracle.tables(st)
    fa = random_cells(st, 10)
    rho = fa.sum(1)
    u = (fa @ xi) / rho[:, None]
    om = 1.37
    ref = fa + om * (textbook_feq(st, rho, u) - fa)
    for eq, zc in DISC_REGIMES:
        fin = fa - w if zc else fa
        out = oracle.collide(st, W.CENTRAL, eq, zc, np.full(len(w), om), fin)
        np.testing.assert_allclose(_abs(out, w, eq, zc), ref, atol=2e-16)


@pytest.mark.parametrize("st", [W.D2Q9, W.D3Q27])
def test_discrete_cumulant_unit_rates_give_feq(st):
    """With every rate one the cumulant collision returns the distribution whose cumulants are
    those of f_eq: on the full stencils that is the textbook f_eq itself."""
    xi, opp, w, M, Minv = oracle.tables(st)
    fa = random_cells(st, 10)
    rho = fa.sum(1)
    u = (fa @ xi) / rho[:, None]
    for zc in (0, 1):
        fin = fa - w if zc else fa
        out = oracle.collide(st, W.CUMULANT, W.EQ_DISCRETE, zc, np.ones(len(w)), fin)
        np.testing.assert_allclose(_abs(out, w, W.EQ_DISCRETE, zc), textbook_feq(st, rho, u), atol=2e-16)


@pytest.mark.parametrize("st", STENCILS)
@pytest.mark.parametrize("space", [W.POPULATION, W.RAW, W.CENTRAL, W.CUMULANT])
def test_discrete_equilibrium_fixed_point_and_conservation(st, space):
    """f_eq is a fixed point of the collision with the discrete equilibrium (any rates), and
    every collision conserves mass and momentum."""
    xi, opp, w, M, Minv = oracle.tables(st)
    rng = np.random.default_rng(4)
    n = 8
    rho = 1 + rng.uniform(-0.05, 0.05, n)
    u = rng.uniform(-0.08, 0.08, (n, 3))
    if W.DIM_OF[st] == 2:
        u[:, 2] = 0
    feq = textbook_feq(st, rho, u)
    fa = random_cells(st, n)
    regimes = [(W.EQ_DISCRETE, 0), (W.EQ_DISCRETE, 1)] + ([] if space == W.CUMULANT else
                                                           [(W.EQ_DISCRETE_DELTA, 1)])
    for eq, zc in regimes:
        rates = rates_for(st, space)
        out = oracle.collide(st, space, eq, zc, rates, feq - w if zc else feq)
        np.testing.assert_allclose(_abs(out, w, eq, zc), feq, atol=3e-16)
        got = oracle.equilibrium(st, space, eq, zc, rho, u)
        np.testing.assert_allclose(_abs(got, w, eq, zc), feq, atol=3e-16)
        out = _abs(oracle.collide(st, space, eq, zc, rates, fa - w if zc else fa), w, eq, zc)
        np.testing.assert_allclose(out.sum(1), fa.sum(1), atol=2e-15)
        np.testing.assert_allclose(out @ xi, fa @ xi, atol=2e-16)


def _acoustic_decay(st, space, eq, zc, om_s, om_b, L=64, steps=700, A=1e-4):
    """Standing longitudinal wave rho = 1 + A cos(k x), u = 0 on an L-periodic box (2D: L x 4,
    3D: L x 2 x 2); returns the amplitude series a(t) / A of the cos(k x) mode of rho."""
    d = W.DIM_OF[st]
    shape = (L, 4, 1) if d == 2 else (L, 2, 2)
    nx, ny, nz = shape
    zz = nz if d == 3 else 1
    x = np.arange(nx)
    k = 2 * math.pi / L
    rho = np.broadcast_to(1 + A * np.cos(k * x), (zz, ny, nx))
    u = np.zeros((rho.size, 3))
    q = W.Q_OF[st]
    feq = oracle.equilibrium(st, space, eq, zc, np.ascontiguousarray(rho).reshape(-1), u)
    sim = oracle.Sim(st, space, eq, zc, W.rates_from_groups(st, {"s": om_s, "b": om_b}), shape, prec=oracle.DOUBLE)
    sim.set(np.ascontiguousarray(feq.T.reshape(q, zz, ny, nx)))
    c = np.cos(k * x)
    amps = np.empty(steps)
    for t in range(steps):
        r, _ = sim.macroscopic()
        amps[t] = ((r.reshape(-1, nx).mean(0) - 1) * c).sum() / (c * c).sum()
        sim.step(1)
    return amps / A


@pytest.mark.parametrize("st,space,eq,zc", [
    (W.D2Q9, W.RAW, W.EQ_DELTA, 1), (W.D2Q9, W.CENTRAL, W.EQ_ABSOLUTE, 1), (W.D2Q9, W.CUMULANT, W.EQ_ABSOLUTE, 1),
    (W.D3Q19, W.RAW, W.EQ_DELTA, 1), (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1),
])
@pytest.mark.parametrize("om_b", [0.8, 1.6])
def test_acoustic_attenuation_pins_bulk_rate(st, space, eq, zc, om_b):
    """The bulk rate (reading R3: omega_b on x^2 + y^2 (+ z^2)) fixes the attenuation of sound.
    Linearised isothermal Navier-Stokes with the viscous stress of the relaxed second moments,
    sigma = rho cs2 [tau_s (S - (2/D) div(u) I) + tau_b (2/D) div(u) I], tau = 1/omega - 1/2,
    gives for a standing wave rho' ~ exp(-Gamma t) (cos(w t) + Gamma / w sin(w t)) with
    Gamma = nu_L k^2 / 2, w^2 = cs2 k^2 - Gamma^2 and the longitudinal viscosity
    nu_L = 2 (D - 1) / D nu + (2 / D) cs2 tau_b (nu = cs2 tau_s).  The fitted Gamma matches
    within 1 % (observed <= 0.05 % at L = 64) for two bulk rates with the shear rate fixed: a
    bulk rate acting on the wrong polynomial group, or not at all, moves Gamma by 3.5x."""
    from scipy.optimize import curve_fit

    cs2, om_s, L, steps = 1 / 3, 1.6, 64, 700
    D = W.DIM_OF[st]
    k = 2 * math.pi / L
    tau_s, tau_b = 1 / om_s - 0.5, 1 / om_b - 0.5
    nu_L = 2 * (D - 1) / D * cs2 * tau_s + 2 / D * cs2 * tau_b
    G0 = nu_L * k * k / 2
    w0 = math.sqrt(cs2 * k * k - G0 * G0)
    a = _acoustic_decay(st, space, eq, zc, om_s, om_b, L, steps)
    model = lambda t, G, w: np.exp(-G * t) * (np.cos(w * t) + G / w * np.sin(w * t))  # noqa: E731
    (G, w), _ = curve_fit(model, np.arange(steps, dtype=np.float64), a, p0=(G0, w0))
    assert abs(G / G0 - 1) < 1e-2, (G, G0)
    assert abs(w / w0 - 1) < 1e-2, (w, w0)


# ------------------------------------------------ WO-MRT basis (reading R31) ---
def hermite_products(stencil, mono):
    """Closed form of the weighted-orthogonal basis on the tensor-product lattices D2Q9 and
    D3Q27: prod_a H_{e_a}(xi_a) with H_0 = 1, H_1 = t, H_2 = t^2 - 1/3 (the 1D D1Q3 weights
    2/3, 1/6, 1/6 make {1, t, t^2 - 1/3} orthogonal; products stay orthogonal)."""
    xi = oracle.tables(stencil)[0].astype(float)
    H = [lambda t: np.ones_like(t), lambda t: t, lambda t: t * t - 1.0 / 3.0]
    rows = []
    for e in mono:
        v = np.ones(xi.shape[0])
        for a in range(3):
            v = v * H[e[a]](xi[:, a])
        rows.append(v)
    return np.array(rows)


@pytest.mark.parametrize("st", [W.D2Q9, W.D3Q27])
def test_wo_basis_is_hermite_on_product_lattices(st):
    M, G, mono = oracle.wo_basis(st)
    # graded-lexicographic order of the documented list (include/lbm.h)
    deg = mono.sum(1)
    assert (np.diff(deg) >= 0).all() and tuple(mono[0]) == (0, 0, 0)
    np.testing.assert_allclose(M, hermite_products(st, mono), atol=1e-15, rtol=0)


def test_wo_basis_d3q19_orthogonal_and_triangular():
    """D3Q19 lacks the corners, so its order-4 polynomials are not Hermite products; pin the
    defining properties: W-orthogonality, monic in the leading monomial (G unit lower
    triangular in graded order), and the orders <= 2 equal to the Hermite products (every
    inner product involved is an odd moment or sum_i w_i xi_x^2 xi_y^2 = 1/9).  From order 3
    on they differ: <x (y^2 - 1/3), x (z^2 - 1/3)> = -1/27 on D3Q19 (no corners)."""
    st = W.D3Q19
    M, G, mono = oracle.wo_basis(st)
    w = oracle.tables(st)[2]
    gram = M @ np.diag(w) @ M.T
    np.testing.assert_allclose(gram - np.diag(np.diag(gram)), 0, atol=1e-16)
    assert (np.diag(gram) > 1e-3).all()
    np.testing.assert_allclose(np.diag(G), 1.0)
    np.testing.assert_allclose(np.triu(G, 1), 0.0)
    low = mono.sum(1) <= 2
    np.testing.assert_allclose(M[low], hermite_products(st, mono)[low], atol=1e-15)
    k = [tuple(e) for e in mono].index((1, 0, 2))  # p = x z^2 - x/3 + (x y^2 - x/3)/2 (hand-derived: <xz^2, p_xy2> / <p_xy2, p_xy2> = (-1/27) / (2/27))
    kk = [tuple(e) for e in mono].index((1, 2, 0))
    assert abs(G[k, kk] - 0.5) < 1e-15
    # D3Q19 x^2 y^2 - projection: <x^2y^2, z^2 - 1/3> = -1/27 != 0, so the z^2 term survives
    k = [tuple(e) for e in mono].index((2, 2, 0))
    kz = [tuple(e) for e in mono].index((0, 0, 2))
    assert abs(G[k, kz]) > 1e-3


@pytest.mark.parametrize("st", STENCILS)
def test_wo_collision_eigenvectors(st):
    """In the weighted-orthogonal basis the collision is diagonal in the W-inner product: the
    non-conserved perturbation delta_k = w o p_k(xi) (it leaves rho and u unchanged) relaxes
    as delta_k -> (1 - omega_k) delta_k, for every regime (PAPER.md:271-319 with T = M_wo).
    D2Q9 / D3Q27: p_k are the Hermite products typed above; D3Q19: the oracle's rows."""
    xi, opp, w, M, Minv = oracle.tables(st)
    Mw, G, mono = oracle.wo_basis(st)
    P = hermite_products(st, mono) if st != W.D3Q19 else Mw
    rates = W.rates_random(st, seed=11)
    rng = np.random.default_rng(4)
    n = 6
    rho = 1 + rng.uniform(-0.04, 0.04, n)
    u = rng.uniform(-0.08, 0.08, (n, 3))
    if W.DIM_OF[st] == 2:
        u[:, 2] = 0
    d = W.DIM_OF[st]
    for eq, zc in [(W.EQ_ABSOLUTE, 0), (W.EQ_DELTA, 1), (W.EQ_ABSOLUTE, 1), (W.EQ_ABSOLUTE_F0, 1)]:
        feq = oracle.equilibrium(st, W.RAW_WO, eq, zc, rho, u)
        np.testing.assert_allclose(oracle.collide(st, W.RAW_WO, eq, zc, rates, feq), feq, atol=1e-16)
        for k in range(1 + d, W.Q_OF[st]):
            delta = 1e-3 * w * P[k]
            out = oracle.collide(st, W.RAW_WO, eq, zc, rates, feq + delta)
            np.testing.assert_allclose(out, feq + (1 - rates[k]) * delta, atol=2e-16, rtol=0,
                                       err_msg=f"eq {eq} zc {zc} polynomial {k} {mono[k]}")


@pytest.mark.parametrize("st", STENCILS)
def test_wo_equal_rates_is_bgk(st):
    """All rates equal: WO-MRT = raw MRT = BGK with the method's truncated-raw f_eq."""
    fa = random_cells(st, 20)
    om = 1.37
    for eq, zc in ALL_REGIMES:
        w = oracle.tables(st)[2]
        fin = fa - w if zc else fa
        a = oracle.collide(st, W.RAW_WO, eq, zc, np.full(W.Q_OF[st], om), fin)
        b = oracle.collide(st, W.POPULATION, eq, zc, [om], fin)
        np.testing.assert_allclose(a, b, atol=2e-16, rtol=0)


def test_wo_tgv_decay_and_regimes():
    """R-WO-MRT on D2Q9 (second-order polynomials at omega_s, the rest 1) decays at
    exp(-4 nu k^2 t) within 1 %, and the literal population-space background
    (LBM_EQ_ABSOLUTE_F0, reading R30) is admitted only with zero-centered storage."""
    st, L, steps, nu = W.D2Q9, 48, 300, 0.05
    om = W.omega_from_nu(nu)
    rho, u = W.tgv_fields(L, L, 1, 0.05)
    for eq, zc in [(W.EQ_DELTA, 1), (W.EQ_ABSOLUTE_F0, 1)]:
        feq = oracle.equilibrium(st, W.RAW_WO, eq, zc, rho.reshape(-1), u.reshape(3, -1).T)
        sim = oracle.Sim(st, W.RAW_WO, eq, zc, W.wo_regularized_rates(st, om), (L, L, 1))
        sim.set(np.ascontiguousarray(feq.T.reshape(9, 1, L, L)))
        r0, u0 = sim.macroscopic()
        e0 = (r0 * (u0 ** 2).sum(0)).sum()
        sim.step(steps)
        r1, u1 = sim.macroscopic()
        ratio = (r1 * (u1 ** 2).sum(0)).sum() / e0
        ref = W.tgv_energy_ratio(nu, L, steps)
        assert abs(ratio / ref - 1) < 1e-2, (eq, ratio, ref)
    with pytest.raises(ValueError):
        oracle.Sim(st, W.CENTRAL, W.EQ_ABSOLUTE_F0, 0, W.rate_set_p(st), (8, 8, 1))


@pytest.mark.parametrize("st", STENCILS)
@pytest.mark.parametrize("space", [W.POPULATION, W.RAW, W.CENTRAL, W.CUMULANT])
def test_background_density_is_a_unit_choice(st, space):
    """rho0 ("typically set to unity"; reading R21): the update is homogeneous of
    degree one in the populations — f_eq(lambda rho, u) = lambda f_eq(rho, u) and
    u = j / rho is scale free (eq:DensityAndVelocity), every transform is
    linear and the cumulants are normalised by rho — so the run with
    background density lambda is lambda times the run with background density one:
    C(lambda f) = lambda C(f).  lambda = 2 is exact in floating point, lambda = 3 to rounding."""
    rng = np.random.default_rng(21)
    n = 24
    rho = rng.uniform(0.9, 1.1, n)
    u = rng.uniform(-0.05, 0.05, (n, 3))
    if st == W.D2Q9:
        u[:, 2] = 0
    f = oracle.equilibrium(st, space, W.EQ_ABSOLUTE, 0, rho, u)
    f = f * (1 + 1e-2 * rng.uniform(-1, 1, f.shape))
    rates = [1.3] if space == W.POPULATION else W.rates_random(st)
    base = oracle.collide(st, space, W.EQ_ABSOLUTE, 0, rates, f)
    np.testing.assert_array_equal(oracle.collide(st, space, W.EQ_ABSOLUTE, 0, rates, 2 * f), 2 * base)
    np.testing.assert_allclose(oracle.collide(st, space, W.EQ_ABSOLUTE, 0, rates, 3 * f), 3 * base,
                               rtol=1e-14, atol=1e-17)
    np.testing.assert_allclose(oracle.equilibrium(st, space, W.EQ_ABSOLUTE, 0, 3 * rho, u),
                               3 * oracle.equilibrium(st, space, W.EQ_ABSOLUTE, 0, rho, u), rtol=1e-15)


@pytest.mark.parametrize("space", [W.CENTRAL, W.CUMULANT])
def test_swe_background_depth_is_a_gravity_rescaling(space):
    """h0 (the shallow-water background depth, reading R33 fixes h0 = 1): Zhou's equilibrium
    (eq:DiscreteShallowWaterEquilibrium) and the Maxwellian at
    cs^2 = g h / 2 satisfy f_eq(lambda h, u; g) = lambda f_eq(h, u; lambda g)
    (every g enters as g h^2 or g h cs-products), so a depth scale lambda is the h0 = 1 run with
    gravity lambda g: C(lambda f; g) = lambda C(f; lambda g)."""
    st, g = W.D2Q9, 0.0613125
    rng = np.random.default_rng(22)
    n = 16
    h = rng.uniform(1.0, 3.0, n)
    u = np.zeros((n, 3))
    u[:, :2] = rng.uniform(-0.05, 0.05, (n, 2))
    lam = 2.0
    np.testing.assert_allclose(oracle.equilibrium(st, space, W.EQ_SWE, 0, lam * h, u, g=g),
                               lam * oracle.equilibrium(st, space, W.EQ_SWE, 0, h, u, g=lam * g), rtol=1e-15,
                               atol=1e-17)
    f = oracle.equilibrium(st, space, W.EQ_SWE, 0, h, u, g=lam * g) * (1 + 1e-2 * rng.uniform(-1, 1, (n, 9)))
    rates = W.rates_random(st)
    np.testing.assert_allclose(oracle.collide(st, space, W.EQ_SWE, 0, rates, lam * f, g=g),
                               lam * oracle.collide(st, space, W.EQ_SWE, 0, rates, f, g=lam * g), rtol=1e-14,
                               atol=1e-16)
