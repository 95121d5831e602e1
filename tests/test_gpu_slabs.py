"""Slab decomposition on one GPU: N contexts (ranks 0..N-1 of N) in one process,
connected by LocalTransport, must reproduce the single-rank run BITWISE
(same per-cell arithmetic; only the ghost-plane plumbing differs), and match
the oracle at full parity."""
from __future__ import annotations

import os

import numpy as np
import pytest

import workloads as W
from gpu_helpers import F64_TOL, gate_error, initial_state, oracle_run, round_to

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2211_02435_b200 import distributed as D  # noqa: E402
from paper_2211_02435_b200 import lbm as L  # noqa: E402


def run_slabs(st, space, eq, zc, rates, shape, f0, steps, nranks, bc=None, streaming=L.LBM_PULL):
    nx, ny, nz = shape
    slab_axis = 2 if W.DIM_OF[st] == 2 else 1  # in the [q][z][y][x] host layout (2D: [q][1][y][x])
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, bc=bc, rank=r, nranks=nranks,
                      streaming=streaming) for r in range(nranks)]
    for lat in lats:
        sl = [slice(None)] * 4
        sl[slab_axis] = slice(lat.offset, lat.offset + lat.extent)
        lat.set_populations(np.ascontiguousarray(f0[tuple(sl)]))
    D.prime_local(lats)
    D.step_local(lats, steps)
    out = np.concatenate([lat.get_populations() for lat in lats], axis=slab_axis)
    for lat in lats:
        lat.close()
    return out


@pytest.mark.parametrize("st,space,eq,zc,nranks", [
    (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, 2),
    (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, 4),
    (W.D3Q19, W.RAW, W.EQ_DELTA, 1, 3),
    (W.D2Q9, W.CENTRAL, W.EQ_ABSOLUTE, 0, 4),
])
def test_slabs_equal_single_rank_bitwise(st, space, eq, zc, nranks):
    shape = (20, 12, 1) if st == W.D2Q9 else (20, 10, 12)
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(20)
        single = lat.get_populations()
    multi = run_slabs(st, space, eq, zc, rates, shape, f0, 20, nranks)
    np.testing.assert_array_equal(multi, single)


def test_slabs_with_walls_match_oracle():
    st, space, eq, zc = W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1
    shape = (16, 10, 16)
    bc = [[0, 0], [0, 0], [L.LBM_BC_NOSLIP, L.LBM_BC_NOSLIP]]
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    multi = run_slabs(st, space, eq, zc, rates, shape, f0, 30, 4, bc=bc)
    ref = oracle_run(st, space, eq, zc, rates, shape, f0, 30, bc=bc)
    assert gate_error(st, multi, ref, zc) < F64_TOL


@pytest.mark.parametrize("st,space,eq,zc,nranks", [
    (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, 2),
    (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, 3),
    (W.D2Q9, W.RAW, W.EQ_DELTA, 1, 4),
])
@pytest.mark.parametrize("steps", [7, 8])
def test_aa_slabs_equal_single_rank_bitwise(st, space, eq, zc, nranks, steps):
    """Multi-rank AA (row f4): the pre-odd / post-odd ghost exchange reproduces the
    single-rank AA run (itself == pull, reading R11) bitwise at both parities."""
    shape = (20, 12, 1) if st == W.D2Q9 else (20, 10, 12)
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        single = lat.get_populations()
    multi = run_slabs(st, space, eq, zc, rates, shape, f0, steps, nranks, streaming=L.LBM_AA)
    np.testing.assert_array_equal(multi, single)


# ----------------------------------------------------------- fused halo push (lbm_peer_*)
def run_slabs_peer(st, space, eq, zc, rates, shape, f0, steps, nranks, bc=None, reprime_at=None,
                   streaming=L.LBM_PULL):
    slab_axis = 2 if W.DIM_OF[st] == 2 else 1
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, bc=bc, rank=r, nranks=nranks,
                      streaming=streaming) for r in range(nranks)]

    def load(f):
        for lat in lats:
            sl = [slice(None)] * 4
            sl[slab_axis] = slice(lat.offset, lat.offset + lat.extent)
            lat.set_populations(np.ascontiguousarray(f[tuple(sl)]))

    load(f0)
    D.connect_local(lats)
    done = 0
    if reprime_at is not None:  # run, reload a state mid-run, prime again, continue
        D.step_peer_local(lats, reprime_at)
        mid = np.concatenate([lat.get_populations() for lat in lats], axis=slab_axis)
        load(mid)
        for lat in lats:
            lat.peer_prime()
        done = reprime_at
    D.step_peer_local(lats, steps - done)
    out = np.concatenate([lat.get_populations() for lat in lats], axis=slab_axis)
    for lat in lats:
        lat.close()
    return out


@pytest.mark.parametrize("st,space,eq,zc,nranks,nz", [
    (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, 2, 12),
    (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, 4, 12),
    (W.D3Q27, W.CENTRAL, W.EQ_DELTA, 1, 3, 6),     # two planes per slab: no interior
    (W.D3Q19, W.RAW, W.EQ_DELTA, 1, 2, 8),
    (W.D2Q9, W.CENTRAL, W.EQ_ABSOLUTE, 0, 4, 1),
])
def test_peer_push_equals_single_rank_bitwise(st, space, eq, zc, nranks, nz):
    """Fused halo push: boundary kernels store into the neighbours' ghost planes, device
    flags order the steps; equals the single-rank run bitwise, incl. a re-prime mid-run."""
    shape = (20, 4 * nranks, 1) if st == W.D2Q9 else (20, 10, nz)
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(13)
        single = lat.get_populations()
    multi = run_slabs_peer(st, space, eq, zc, rates, shape, f0, 13, nranks, reprime_at=5)
    np.testing.assert_array_equal(multi, single)


@pytest.mark.parametrize("fence", ["0", "1", "2"])
def test_peer_push_with_walls_matches_oracle(fence, monkeypatch):
    monkeypatch.setenv("LBM_PEER_FENCE", fence)  # per-thread system fence after the pushes
    st, space, eq, zc = W.D3Q27, W.RAW, W.EQ_DELTA, 1
    shape = (16, 10, 16)
    bc = [[0, 0], [L.LBM_BC_NOSLIP, L.LBM_BC_NOSLIP], [L.LBM_BC_NOSLIP, L.LBM_BC_NOSLIP]]
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    multi = run_slabs_peer(st, space, eq, zc, rates, shape, f0, 25, 4, bc=bc)
    ref = oracle_run(st, space, eq, zc, rates, shape, f0, 25, bc=bc)
    assert gate_error(st, multi, ref, zc) < F64_TOL


def test_peer_rejects_mismatched_ring():
    st, space, eq, zc = W.D3Q19, W.RAW, W.EQ_DELTA, 1
    rates = W.rate_set_p(st)
    a = L.Lattice(st, space, eq, rates, (16, 8, 8), rank=0, nranks=2)
    b = L.Lattice(st, space, eq, rates, (16, 8, 8), rank=1, nranks=2)
    c = L.Lattice(st, space, eq, rates, (16, 8, 16), rank=1, nranks=2)
    ia, ib, ic = a.peer_export(), b.peer_export(), c.peer_export()
    with pytest.raises(L.LbmError):
        a.peer_connect(ic, ic)  # other lattice
    with pytest.raises(L.LbmError):
        a.peer_connect(ia, ia)  # wrong ranks
    a.peer_connect(ib, ib)
    with L.Lattice(st, space, eq, rates, (16, 8, 8)) as d:  # one rank: nothing to connect
        with pytest.raises(L.LbmError):
            d.peer_export()
    for x in (a, b, c):
        x.close()


# ----------------------------------------------------------- SURVEY.md 8(d) multi-rank parity runs
def tgv_state(st, space, eq, zc, shape, lat):
    rho, u = W.tgv_fields(shape[0], shape[1], shape[2], 0.05)
    lat.init_macroscopic(np.ascontiguousarray(rho), np.ascontiguousarray(u[:lat.d]))
    return lat.get_populations()


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_c4_multirank_64cubed_bitwise(nranks):
    """C4 (D3Q27 cumulant, zc + eq, fp64, pull) at 64^3, 100 steps, N = 2, 4, 8 slab ranks
    (8-plane slabs at N = 8) with the fused halo push and with the exchange: both equal the
    single-rank run bitwise (the single-rank run itself matches the oracle:
    test_gpu_parity.py::test_config4_d3q27_cumulant)."""
    st, space, eq, zc = W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1
    shape = (64, 64, 64)
    rates = W.rate_set_p(st)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        f0 = initial_state(st, space, eq, zc, shape)
        lat.set_populations(f0)
        lat.step(100)
        single = lat.get_populations()
    np.testing.assert_array_equal(run_slabs_peer(st, space, eq, zc, rates, shape, f0, 100, nranks), single)
    np.testing.assert_array_equal(run_slabs(st, space, eq, zc, rates, shape, f0, 100, nranks), single)


def test_c4_eight_slabs_256cubed_bitwise():
    """The N = 8 decomposition of a 256^3 C4 lattice (32-plane slabs, fused halo push)
    reproduces the single-rank run bitwise after 20 steps."""
    st, space, eq, zc = W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1
    shape = (256, 256, 256)
    rates = W.rate_set_p(st)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        f0 = tgv_state(st, space, eq, zc, shape, lat)
        lat.step(20)
        single = lat.get_populations()
    np.testing.assert_array_equal(run_slabs_peer(st, space, eq, zc, rates, shape, f0, 20, 8), single)


def test_c5_eight_slabs_128squared():
    """C5 (D2Q9 shallow water, CM, Zhou eq., absolute, fp64) at 128^2, dam radius 8, 100
    steps: N = 8 y-slabs (fused halo push) equal the single-rank run bitwise, which matches
    the oracle (cell-normalised metric, reading R12b)."""
    st, space, eq, zc = W.D2Q9, W.CENTRAL, W.EQ_SWE, 0
    shape = (128, 128, 1)
    g, nu, om = W.swe_lattice_parameters()
    rates = W.regularized_rates(st, om)
    f0 = initial_state(st, space, eq, zc, shape, g=g, noise=0.0, dam=(8.0, 6.25, 1.25))
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, swe_g=g) as lat:
        lat.set_populations(f0)
        lat.step(100)
        single = lat.get_populations()
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, swe_g=g, rank=r, nranks=8) for r in range(8)]
    for lat in lats:
        lat.set_populations(np.ascontiguousarray(f0[:, :, lat.offset:lat.offset + lat.extent]))
    D.connect_local(lats)
    D.step_peer_local(lats, 100)
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=2)
    for lat in lats:
        lat.close()
    np.testing.assert_array_equal(multi, single)
    ref = oracle_run(st, space, eq, zc, rates, shape, f0, 100, g=g)
    assert gate_error(st, single, ref, zc, norm="cell") < F64_TOL


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_peer_push_graph_replay_bitwise(graphs, monkeypatch):
    """Whole lbm_step_peer(n) calls per context (not interleaved step by step; one host thread
    per context) equal the single-rank run.  On one GPU the phases are host-ordered (no graphs);
    with one GPU per rank n >= 32 replays captured graphs (test_peer_device_waits_across_gpus)."""
    monkeypatch.setenv("LBM_CUDA_GRAPHS", graphs)
    st, space, eq, zc = W.D3Q19, W.CENTRAL, W.EQ_DELTA, 1
    shape, nranks = (24, 10, 12), 3
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(40 + 71)
        single = lat.get_populations()
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=nranks) for r in range(nranks)]
    for lat in lats:
        lat.set_populations(np.ascontiguousarray(f0[:, lat.offset:lat.offset + lat.extent]))
    D.connect_local(lats)
    for n in (40, 71):
        D.on_ranks(lats, lambda lat: lat.step_peer(n))
    for lat in lats:
        lat.sync()
        assert not lat.peer_timed_out()
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=1)
    for lat in lats:
        lat.close()
    np.testing.assert_array_equal(multi, single)


@pytest.mark.parametrize("st,space,eq,zc,nranks", [
    (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, 2),
    (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, 3),
    (W.D3Q19, W.RAW, W.EQ_DELTA, 1, 4),
    (W.D2Q9, W.CUMULANT, W.EQ_ABSOLUTE, 1, 4),
])
@pytest.mark.parametrize("steps,reprime", [(7, None), (8, None), (9, 4), (10, 3)])
def test_peer_aa_equals_single_rank_bitwise(st, space, eq, zc, nranks, steps, reprime):
    """Multi-rank AA with the fused peer path: the odd step's boundary kernels access the
    neighbours' boundary planes directly (no ghost exchange); the canonical state read at
    either parity (odd counts: refreshed ghost planes), incl. a reload + re-prime at both
    parities, equals the single-rank run bitwise."""
    shape = (20, 12, 1) if st == W.D2Q9 else (20, 10, 12)
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        single = lat.get_populations()
    multi = run_slabs_peer(st, space, eq, zc, rates, shape, f0, steps, nranks, reprime_at=reprime,
                           streaming=L.LBM_AA)
    np.testing.assert_array_equal(multi, single)


def test_peer_aa_graph_replay_and_macroscopic():
    """AA peer loop in whole calls per context (captured graphs with one GPU per rank; host-
    ordered phases on one GPU), then the macroscopic fields and the diagnostics at the odd parity match the single-rank run."""
    st, space, eq, zc = W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1
    shape, nranks = (24, 10, 12), 3
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, streaming=L.LBM_AA) as lat:
        lat.set_populations(f0)
        lat.step(33 + 32)
        rho1, u1 = lat.get_macroscopic()
        f1 = lat.get_populations()
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=nranks, streaming=L.LBM_AA)
            for r in range(nranks)]
    for lat in lats:
        lat.set_populations(np.ascontiguousarray(f0[:, lat.offset:lat.offset + lat.extent]))
    D.connect_local(lats)
    for n in (33, 32):
        D.on_ranks(lats, lambda lat: lat.step_peer(n))
    for lat in lats:
        lat.sync()
        assert not lat.peer_timed_out()
    rho = np.concatenate([lat.get_macroscopic()[0] for lat in lats], axis=0)
    u = np.concatenate([lat.get_macroscopic()[1] for lat in lats], axis=1)
    f = np.concatenate([lat.get_populations() for lat in lats], axis=1)
    for lat in lats:
        lat.close()
    np.testing.assert_array_equal(f, f1)
    np.testing.assert_array_equal(rho, rho1)
    np.testing.assert_array_equal(u, u1)


@pytest.mark.parametrize("streaming,space,eq,model", [
    (L.LBM_PULL, W.CENTRAL, W.EQ_DELTA, L.LBM_FORCE_HE),
    (L.LBM_PULL, W.CUMULANT, W.EQ_ABSOLUTE, L.LBM_FORCE_GUO),
    (L.LBM_AA, W.RAW, W.EQ_ABSOLUTE, L.LBM_FORCE_GUO),
])
def test_peer_forced_then_disconnect_equals_single_rank(streaming, space, eq, model):
    """Body forces (He, cumulant first-order source) through the fused peer path, then
    lbm_peer_connect(NULL, NULL) on every rank and more steps through the exchange path
    (lbm_step_region + LocalTransport): the whole run equals the single-rank one bitwise."""
    st, zc, nranks = W.D3Q27, 1, 3
    shape = (20, 10, 12)
    rates = W.rate_set_p(st)
    F = np.array([2e-4, -1e-4, 3e-4])
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, streaming=streaming) as lat:
        lat.set_populations(f0)
        lat.set_force(F, model=model)
        lat.step(9 + 6)
        single = lat.get_populations()
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=nranks, streaming=streaming)
            for r in range(nranks)]
    for lat in lats:
        lat.set_populations(np.ascontiguousarray(f0[:, lat.offset:lat.offset + lat.extent]))
        lat.set_force(F, model=model)
    D.connect_local(lats)
    D.step_peer_local(lats, 9)
    mid = np.concatenate([lat.get_populations() for lat in lats], axis=1)
    for lat in lats:
        lat.sync()
        lat.peer_disconnect()
    for lat in lats:  # reload the canonical state and continue on the exchange path
        lat.set_populations(np.ascontiguousarray(mid[:, lat.offset:lat.offset + lat.extent]))
    D.prime_local(lats)
    D.step_local(lats, 6)
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=1)
    for lat in lats:
        lat.close()
    np.testing.assert_array_equal(multi, single)


@pytest.mark.parametrize("st,space,eq,zc,prec,shape,nranks", [
    (W.D3Q19, W.RAW, W.EQ_DELTA, 1, L.LBM_FP64, (32, 16, 24), 2),
    (W.D3Q19, W.CENTRAL, W.EQ_ABSOLUTE, 1, L.LBM_FP64, (32, 16, 24), 3),
    (W.D3Q19, W.RAW, W.EQ_DELTA, 1, L.LBM_FP32, (32, 16, 24), 4),
    (W.D3Q27, W.RAW, W.EQ_DELTA, 1, L.LBM_FP64, (32, 16, 18), 3),
    (W.D2Q9, W.CENTRAL, W.EQ_SWE, 0, L.LBM_FP64, (256, 36, 1), 3),
    (W.D2Q9, W.POPULATION, W.EQ_DELTA, 1, L.LBM_FP64, (256, 24, 1), 4),
])
def test_peer_two_step_sweeps_match_single_rank(st, space, eq, zc, prec, shape, nranks, monkeypatch):
    """Temporal blocking across ranks on the peer path: interior planes by the two-step sweep,
    the boundary regions by two single steps through the scratch planes with pushes into the
    neighbours' scratch and ghost planes; pairs plus a trailing single step match the
    single-rank run to rounding and the oracle at full parity."""
    monkeypatch.setenv("LBM_PEER_TB", "1")  # small lattices: pairs despite < 2 waves of CTAs
    monkeypatch.setenv("LBM_TB_DEPTH", "2")  # 2D slabs would otherwise advance triples
    g = W.swe_lattice_parameters()[0] if eq == W.EQ_SWE else 0.0
    rates = W.rate_set_p(st) if space != W.POPULATION else [1.3]
    if eq == W.EQ_SWE:
        f0 = initial_state(st, space, eq, zc, shape, g=g, noise=0.0, dam=(8.0, 6.25, 1.25))
    else:
        f0 = round_to(initial_state(st, space, eq, zc, shape), prec)
    steps = 9
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, precision=prec, swe_g=g) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        single = lat.get_populations()
    slab_axis = 2 if W.DIM_OF[st] == 2 else 1
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, precision=prec, swe_g=g, rank=r,
                      nranks=nranks) for r in range(nranks)]
    for lat in lats:
        sl = [slice(None)] * 4
        sl[slab_axis] = slice(lat.offset, lat.offset + lat.extent)
        lat.set_populations(np.ascontiguousarray(f0[tuple(sl)]))
    D.connect_local(lats)
    assert all(lat.info().temporal_blocking == 2 for lat in lats)
    D.step_peer_local(lats, steps, chunk=2)
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=slab_axis)
    for lat in lats:
        lat.close()
    norm = "cell" if eq == W.EQ_SWE else "population"
    tol = 1e-13 if prec == L.LBM_FP64 else 2e-6
    assert gate_error(st, multi, single, zc, norm=norm) < tol
    if prec == L.LBM_FP64:
        ref = oracle_run(st, space, eq, zc, rates, shape, f0, steps, g=g)
        assert gate_error(st, multi, ref, zc, norm=norm) < F64_TOL


def test_peer_two_step_sweeps_graph_replay(monkeypatch):
    """Two-step sweeps across ranks in whole calls (inside captured 32-step graphs, 16 pairs per
    graph, with one GPU per rank; host-ordered phases on one GPU) plus a remainder of pairs and a single step: equal to the single-rank run to rounding."""
    monkeypatch.setenv("LBM_PEER_TB", "1")
    st, space, eq, zc = W.D3Q19, W.RAW, W.EQ_DELTA, 1
    shape, nranks, steps = (32, 16, 24), 2, 71
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        single = lat.get_populations()
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=nranks) for r in range(nranks)]
    for lat in lats:
        lat.set_populations(np.ascontiguousarray(f0[:, lat.offset:lat.offset + lat.extent]))
    D.connect_local(lats)
    for chunk in (64, 7):  # two graph replays per context, then 3 pairs + 1 single step
        D.on_ranks(lats, lambda lat: lat.step_peer(chunk))
    for lat in lats:
        lat.sync()
        assert not lat.peer_timed_out()
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=1)
    for lat in lats:
        lat.close()
    assert gate_error(st, multi, single, zc) < 1e-13


@pytest.mark.parametrize("st,space,eq,zc,shape,nranks", [
    (W.D3Q19, W.RAW, W.EQ_DELTA, 1, (32, 16, 24), 2),
    (W.D3Q19, W.CUMULANT, W.EQ_ABSOLUTE, 1, (32, 16, 24), 4),
    (W.D2Q9, W.CENTRAL, W.EQ_ABSOLUTE, 1, (256, 36, 1), 3),
])
def test_exchange_path_two_step_regions(st, space, eq, zc, shape, nranks, monkeypatch):
    """Two-step sweeps across ranks with an external exchange (LBM_REGION_PAIR_* +
    lbm_get_halo(2), the SlabRunner sequence with LocalTransport): pairs plus a single step
    equal the single-rank run to rounding and the oracle at the gate."""
    monkeypatch.setenv("LBM_PEER_TB", "1")
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    steps = 9
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        single = lat.get_populations()
    slab_axis = 2 if W.DIM_OF[st] == 2 else 1
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=nranks) for r in range(nranks)]
    for lat in lats:
        sl = [slice(None)] * 4
        sl[slab_axis] = slice(lat.offset, lat.offset + lat.extent)
        lat.set_populations(np.ascontiguousarray(f0[tuple(sl)]))
    assert all(D.supports_pairs(lat) for lat in lats)
    D.prime_local(lats)
    D.step_local(lats, steps, pairs=True)
    assert lats[0].info().steps_done == steps
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=slab_axis)
    for lat in lats:
        lat.close()
    assert gate_error(st, multi, single, zc) < 1e-13
    assert gate_error(st, multi, oracle_run(st, space, eq, zc, rates, shape, f0, steps), zc) < F64_TOL


def test_peer_waits_are_host_ordered_when_ranks_share_a_gpu(monkeypatch):
    """Contexts whose neighbours share their GPU never launch a kernel that spins on another
    rank's flag (B200_PROFILING: such launches on one GPU are not co-scheduled); the host polls
    the flags instead (lbm_info.peer_wait_host), no graphs.  LBM_PEER_WAIT overrides at connect."""
    st, space, eq, zc = W.D3Q19, W.RAW, W.EQ_DELTA, 1
    shape = (16, 8, 12)
    rates = W.rate_set_p(st)
    for env, want in ((None, 1), ("device", 0), ("host", 1)):
        if env is None:
            monkeypatch.delenv("LBM_PEER_WAIT", raising=False)
        else:
            monkeypatch.setenv("LBM_PEER_WAIT", env)
        lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=2, device=0)
                for r in range(2)]
        infos = [lat.peer_export() for lat in lats]
        for r, lat in enumerate(lats):
            lo, hi = D.neighbours(r, 2)
            lat.peer_connect(infos[lo], infos[hi])
        assert [lat.info().peer_wait_host for lat in lats] == [want, want]
        for lat in lats:
            lat.close()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="device-side peer waits need one GPU per rank")
@pytest.mark.parametrize("tb,st", [("0", W.D3Q19), ("1", W.D3Q19), ("1", W.D2Q9)])
def test_peer_device_waits_across_gpus(tb, st, monkeypatch):
    """The deployment case: every context on its own GPU (in one process), device-side waits,
    n >= 32 steps from captured graphs, single steps, two-step pairs (3D) and triples (2D, 36-step
    graphs); equal to the single rank (bitwise for single steps, to rounding when fused)."""
    monkeypatch.setenv("LBM_PEER_TB", tb)
    monkeypatch.delenv("LBM_PEER_WAIT", raising=False)
    space, eq, zc = W.RAW, W.EQ_DELTA, 1
    ndev = torch.cuda.device_count()
    nranks = min(ndev, 4)
    shape, steps = ((256, 12 * nranks, 1) if st == W.D2Q9 else (32, 16, 8 * nranks)), 71
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        single = lat.get_populations()
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=nranks, device=r)
            for r in range(nranks)]
    ax = 2 if st == W.D2Q9 else 1
    for lat in lats:
        sl = [slice(None)] * 4
        sl[ax] = slice(lat.offset, lat.offset + lat.extent)
        lat.set_populations(np.ascontiguousarray(f0[tuple(sl)]))
    D.connect_local(lats)
    assert all(lat.info().peer_wait_host == 0 for lat in lats)
    for chunk in (64, 7):
        for lat in lats:
            lat.step_peer(chunk)
    for lat in lats:
        lat.sync()
        assert not lat.peer_timed_out()
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=ax)
    for lat in lats:
        lat.close()
    if tb == "0":
        np.testing.assert_array_equal(multi, single)
    else:
        assert gate_error(st, multi, single, zc) < 1e-13


def _random_slab_config(k):
    rng = np.random.default_rng(7000 + k)
    st = [W.D2Q9, W.D3Q19, W.D3Q27][rng.integers(3)]
    space = [W.POPULATION, W.RAW, W.CENTRAL, W.CUMULANT][rng.integers(4)]
    regimes = [(W.EQ_ABSOLUTE, 0), (W.EQ_ABSOLUTE, 1)] + ([] if space == W.CUMULANT else [(W.EQ_DELTA, 1)])
    eq, zc = regimes[rng.integers(len(regimes))]
    streaming = [L.LBM_PULL, L.LBM_AA][rng.integers(2)]
    transport = ["peer", "exchange"][rng.integers(2)]
    nranks = int(rng.integers(2, 5))
    per = max(int(rng.integers(2, 15)), -(-4 // nranks))  # planes per slab (even split, >= 2; extents >= 4)
    d = W.DIM_OF[st]
    shape = ((256 if rng.random() < 0.5 else int(rng.integers(9, 40)), nranks * per, 1) if d == 2 else
             (int(rng.integers(9, 30)), int(rng.integers(5, 14)), nranks * per))
    pairs = streaming == L.LBM_PULL and rng.random() < 0.5
    steps = int(rng.integers(3, 10))
    return st, space, eq, zc, streaming, transport, nranks, shape, pairs, steps


@pytest.mark.parametrize("k", range(int(os.environ.get("LBM_TEST_DRAWS_MULTI", "40"))))
def test_random_multi_rank_sweep(k, monkeypatch):
    """Seeded random multi-rank draws (stencil, collision space, regime, pull / AA, fused peer
    push or the exchange building blocks, 2-4 ranks, slabs of 2-14 planes, two-step
    sweeps across ranks or single steps) against the single-rank run: bitwise with single
    steps, to rounding with pairs of steps."""
    st, space, eq, zc, streaming, transport, nranks, shape, pairs, steps = _random_slab_config(k)
    monkeypatch.setenv("LBM_PEER_TB", "1" if pairs else "0")
    rates = np.array([1.37]) if space == W.POPULATION else W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape, seed=W.SEED + 11 * k)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, streaming=streaming) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        single = lat.get_populations()
    slab_axis = 2 if W.DIM_OF[st] == 2 else 1
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=nranks, streaming=streaming)
            for r in range(nranks)]
    for lat in lats:
        sl = [slice(None)] * 4
        sl[slab_axis] = slice(lat.offset, lat.offset + lat.extent)
        lat.set_populations(np.ascontiguousarray(f0[tuple(sl)]))
    used_pairs = pairs and all(D.supports_pairs(l) for l in lats)
    if transport == "peer":
        D.connect_local(lats)
        D.step_peer_local(lats, steps, chunk=steps if pairs else 1)
        used_pairs = used_pairs and all(l.info().temporal_blocking >= 2 for l in lats)
    else:
        D.prime_local(lats)
        D.step_local(lats, steps, pairs=pairs)
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=slab_axis)
    for lat in lats:
        lat.close()
    what = (st, space, eq, zc, streaming, transport, nranks, shape, pairs, steps)
    if used_pairs:
        assert gate_error(st, multi, single, zc) < 1e-13, what
    else:
        np.testing.assert_array_equal(multi, single, err_msg=str(what))


@pytest.mark.parametrize("space,eq,zc,prec,nranks,rows,steps", [
    (W.CENTRAL, W.EQ_SWE, 0, L.LBM_FP64, 2, 12, 9),
    (W.CUMULANT, W.EQ_SWE, 1, L.LBM_FP64, 3, 10, 11),
    (W.CENTRAL, W.EQ_ABSOLUTE, 1, L.LBM_FP64, 4, 16, 8),
    (W.RAW, W.EQ_DELTA, 1, L.LBM_FP32, 2, 20, 7),
    (W.POPULATION, W.EQ_DELTA, 1, L.LBM_FP64, 3, 11, 36 + 5),
])
def test_peer_three_step_sweeps_2d_match_single_rank(space, eq, zc, prec, nranks, rows, steps, monkeypatch):
    """2D slabs on the fused peer push advance TRIPLES of steps (interior rows by the depth-3
    sweep, boundary regions by three single steps through the level-1 / level-2 scratch with
    pushes into the neighbours' ghost rows; lbm_info.temporal_blocking == 3), then a pair or a
    single step: equal to the single-rank run to rounding and to the oracle."""
    monkeypatch.setenv("LBM_PEER_TB", "1")
    st = W.D2Q9
    shape = (256, rows * nranks, 1)
    g = W.swe_lattice_parameters()[0] if eq == W.EQ_SWE else 0.0
    rates = (W.regularized_rates(st, W.swe_lattice_parameters()[2]) if eq == W.EQ_SWE else
             (np.array([1.37]) if space == W.POPULATION else W.rate_set_p(st)))
    if eq == W.EQ_SWE:
        f0 = initial_state(st, space, eq, zc, shape, g=g, noise=0.0, dam=(60.0, 6.25, 1.25))
    else:
        f0 = round_to(initial_state(st, space, eq, zc, shape), prec)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, precision=prec, swe_g=g) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        single = lat.get_populations()
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, precision=prec, swe_g=g, rank=r,
                      nranks=nranks) for r in range(nranks)]
    for lat in lats:
        lat.set_populations(np.ascontiguousarray(f0[:, :, lat.offset:lat.offset + lat.extent]))
    D.connect_local(lats)
    assert all(lat.info().temporal_blocking == 3 for lat in lats)
    D.on_ranks(lats, lambda lat: lat.step_peer(steps))
    for lat in lats:
        lat.sync()
        assert not lat.peer_timed_out()
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=2)
    for lat in lats:
        lat.close()
    norm = "cell" if eq == W.EQ_SWE else "population"
    tol = 1e-13 if prec == L.LBM_FP64 else 2e-6
    assert gate_error(st, multi, single, zc, norm=norm) < tol
    if prec == L.LBM_FP64 and eq != W.EQ_SWE:
        ref = oracle_run(st, space, eq, zc, rates, shape, f0, steps, g=g)
        assert gate_error(st, multi, ref, zc) < F64_TOL


@pytest.mark.parametrize("nranks,rows,steps", [(2, 12, 9), (3, 10, 11), (4, 14, 7)])
def test_exchange_three_step_regions_2d(nranks, rows, steps, monkeypatch):
    """The external-exchange building blocks for triples (LBM_REGION_TRIPLE_*, lbm_get_halo(3/4)
    level scratch halos) driven by the in-process transport: equal to the single-rank run to
    rounding."""
    monkeypatch.setenv("LBM_PEER_TB", "1")
    st, space, eq, zc = W.D2Q9, W.CENTRAL, W.EQ_ABSOLUTE, 1
    shape = (256, rows * nranks, 1)
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        single = lat.get_populations()
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=nranks) for r in range(nranks)]
    for lat in lats:
        lat.set_populations(np.ascontiguousarray(f0[:, :, lat.offset:lat.offset + lat.extent]))
    assert all(D.supports_triples(l) and l.info().temporal_blocking == 3 for l in lats)
    D.prime_local(lats)
    D.step_local(lats, steps, pairs=True)
    multi = np.concatenate([lat.get_populations() for lat in lats], axis=2)
    assert all(lat.info().steps_done == steps for lat in lats)
    for lat in lats:
        lat.close()
    assert gate_error(st, multi, single, zc) < 1e-13
