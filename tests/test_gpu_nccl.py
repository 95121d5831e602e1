"""The library's own collective lbm_step over ranks: the in-library
NCCL halo exchange (lbm_domain.nccl_id) and the fused peer push reached through lbm_step.

One GPU per rank is NCCL's rule (two ranks on one device are refused), so on a one-GPU box
the NCCL path runs as ONE rank exchanging with itself: the periodic wrap along the slab axis
goes through the ghost planes and an ncclSend/ncclRecv group per step, exactly the sequence
of every rank of a decomposition (neighbour = itself).  It must equal the plain single-rank
run bitwise (same kernels; only the plumbing differs), and to rounding with the two-step
sweeps (the pair sequence with two exchanges per pair)."""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W
from gpu_helpers import F64_TOL, gate_error, initial_state, oracle_run

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2211_02435_b200 import distributed as D  # noqa: E402
from paper_2211_02435_b200 import lbm as L  # noqa: E402


def single_rank(st, space, eq, zc, rates, shape, f0, steps, **kw):
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, **kw) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        return lat.get_populations()


@pytest.mark.parametrize("st,space,eq,zc,streaming,steps", [
    (W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, L.LBM_PULL, 13),
    (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, L.LBM_AA, 13),
    (W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, L.LBM_AA, 12),
    (W.D2Q9, W.CENTRAL, W.EQ_SWE, 0, L.LBM_PULL, 11),
    (W.D3Q19, W.RAW, W.EQ_DELTA, 1, L.LBM_PULL, 10),
])
def test_nccl_self_exchange_equals_single_rank_bitwise(st, space, eq, zc, streaming, steps):
    shape = (20, 12, 1) if st == W.D2Q9 else (20, 10, 12)
    g = W.swe_lattice_parameters()[0] if eq == W.EQ_SWE else 0.0
    rates = W.regularized_rates(st, 1.3) if eq == W.EQ_SWE else W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape, g=g, noise=0.0 if eq == W.EQ_SWE else 1e-3,
                       **({"dam": (4.0, 6.25, 1.25)} if eq == W.EQ_SWE else {}))
    ref = single_rank(st, space, eq, zc, rates, shape, f0, steps, streaming=streaming, swe_g=g)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, streaming=streaming, swe_g=g,
                   nccl_id=L.nccl_get_unique_id()) as lat:
        lat.set_populations(f0)
        lat.step(5)  # the first call exchanges the current halo (prime) before stepping
        lat.step(steps - 5)
        assert lat.info().steps_done == steps
        got = lat.get_populations()
    np.testing.assert_array_equal(got, ref)


def test_nccl_self_exchange_two_step_sweeps(monkeypatch):
    """Pairs of steps across the NCCL exchange (interior sweep + two boundary steps through the
    scratch planes, two exchanges per pair) plus a trailing single step: to rounding against
    the single-rank run, at the gate against the oracle."""
    monkeypatch.setenv("LBM_PEER_TB", "1")  # small lattice: pairs despite < 2 waves of CTAs
    st, space, eq, zc = W.D3Q19, W.RAW, W.EQ_DELTA, 1
    shape, steps = (32, 16, 24), 9
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    ref = single_rank(st, space, eq, zc, rates, shape, f0, steps)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, nccl_id=L.nccl_get_unique_id()) as lat:
        assert lat.info().temporal_blocking == 2
        lat.set_populations(f0)
        lat.step(steps)
        got = lat.get_populations()
    assert gate_error(st, got, ref, zc) < 1e-13
    assert gate_error(st, got, oracle_run(st, space, eq, zc, rates, shape, f0, steps), zc) < F64_TOL


def test_nccl_re_init_and_macroscopic():
    """lbm_init_macroscopic resets the state; the next lbm_step primes the halo again."""
    st, space, eq, zc = W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1
    shape = (16, 8, 10)
    rates = W.rate_set_p(st)
    rho, u = W.tgv_fields(*shape, 0.05, plane="xz")
    outs = []
    for nid in (None, L.nccl_get_unique_id()):
        with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, nccl_id=nid) as lat:
            for _ in range(2):
                lat.init_macroscopic(rho, u)
                lat.step(7)
            outs.append(lat.get_macroscopic())
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


def test_multi_rank_lbm_step_without_transport_is_unsupported():
    st = W.D3Q27
    with L.Lattice(st, W.CUMULANT, W.EQ_ABSOLUTE, W.rate_set_p(st), (16, 8, 8), rank=0, nranks=2) as lat:
        with pytest.raises(L.LbmError) as e:
            lat.step(1)
        assert e.value.status == L.LBM_EUNSUPPORTED


@pytest.mark.parametrize("streaming", [L.LBM_PULL, L.LBM_AA])
def test_lbm_step_on_peer_connected_contexts_primes_itself(streaming):
    """lbm_step on connected contexts is the fused peer push (lbm_step_peer); after a reload
    mid-run the next lbm_step re-primes by itself (no explicit lbm_peer_prime)."""
    st, space, eq, zc = W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1
    shape, nranks, steps = (20, 10, 12), 3, 11
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    ref = single_rank(st, space, eq, zc, rates, shape, f0, steps)
    lats = [L.Lattice(st, space, eq, rates, shape, zero_centered=zc, rank=r, nranks=nranks, streaming=streaming)
            for r in range(nranks)]

    def load(f):
        for lat in lats:
            lat.set_populations(np.ascontiguousarray(f[:, lat.offset:lat.offset + lat.extent]))

    load(f0)
    infos = [lat.peer_export() for lat in lats]
    for r, lat in enumerate(lats):
        lo, hi = D.neighbours(r, nranks)
        lat.peer_connect(infos[lo], infos[hi])
    for lat in lats:
        lat.sync()
    D.step_peer_local(lats, 4)
    mid = np.concatenate([lat.get_populations() for lat in lats], axis=1)
    load(mid)
    D.step_peer_local(lats, steps - 4)
    got = np.concatenate([lat.get_populations() for lat in lats], axis=1)
    for lat in lats:
        lat.close()
    np.testing.assert_array_equal(got, ref)


def test_device_allocator_hook():
    """lbm_domain.dev_alloc / dev_free: the grids come from the caller's allocator (here the
    torch caching allocator) and are handed back at lbm_destroy."""
    st, space, eq, zc = W.D3Q19, W.RAW, W.EQ_DELTA, 1
    shape = (20, 10, 12)
    rates = W.rate_set_p(st)
    f0 = initial_state(st, space, eq, zc, shape)
    ref = single_rank(st, space, eq, zc, rates, shape, f0, 6)
    live = {}

    def alloc(n):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        live[t.data_ptr()] = t
        return t.data_ptr()

    def free(p):
        live.pop(p)

    lat = L.Lattice(st, space, eq, rates, shape, zero_centered=zc, allocator=(alloc, free))
    assert len(live) == 2  # two pull grids
    lat.set_populations(f0)
    lat.step(6)
    np.testing.assert_array_equal(lat.get_populations(), ref)
    lat.close()
    assert not live


@pytest.mark.parametrize("space,eq,zc,steps", [(W.CENTRAL, W.EQ_SWE, 0, 10), (W.RAW, W.EQ_DELTA, 1, 8)])
def test_nccl_self_exchange_three_step_sweeps_2d(space, eq, zc, steps, monkeypatch):
    """2D triples across the NCCL exchange (interior depth-3 sweep + three boundary steps through
    the level-1 / level-2 scratch, an exchange after each level) plus a trailing single step or
    pair: to rounding against the single-rank run."""
    monkeypatch.setenv("LBM_PEER_TB", "1")
    st, shape = W.D2Q9, (256, 24, 1)
    g = W.swe_lattice_parameters()[0] if eq == W.EQ_SWE else 0.0
    rates = W.regularized_rates(st, W.swe_lattice_parameters()[2]) if eq == W.EQ_SWE else W.rate_set_p(st)
    if eq == W.EQ_SWE:
        f0 = initial_state(st, space, eq, zc, shape, g=g, noise=0.0, dam=(60.0, 6.25, 1.25))
    else:
        f0 = initial_state(st, space, eq, zc, shape)
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, swe_g=g) as lat:
        lat.set_populations(f0)
        lat.step(steps)
        ref = lat.get_populations()
    with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, swe_g=g, nccl_id=L.nccl_get_unique_id()) as lat:
        assert lat.info().temporal_blocking == 3
        lat.set_populations(f0)
        lat.step(steps)
        got = lat.get_populations()
    assert gate_error(st, got, ref, zc, norm="cell" if eq == W.EQ_SWE else "population") < 1e-13
