"""Multi-rank slab plumbing on CPU (gloo, world size 2 and 4): the halo exchange of
paper_2211_02435_b200.distributed moves exactly the slab-crossing population
blocks of the library's device grid layout (lbm_grid_layout) into the neighbours'
ghost planes, with periodic wrap along the slab axis."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2211_02435_b200 as P
from paper_2211_02435_b200 import distributed as D
from paper_2211_02435_b200 import lbm as L


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fill_value(zg, i, y, x):
    """Code of population i at global slab plane zg, row y, column x."""
    return zg * 1e6 + i * 1e4 + y * 1e2 + x


def make_grid(stencil, prec, shape, rank, nranks):
    """A rank's grid in the device layout with interior planes coded by global position."""
    lay = P.grid_layout(stencil, prec, shape, nranks)
    nx, ny, nz = shape
    two_d = stencil == L.LBM_D2Q9
    slab = ny if two_d else nz
    nyy = 1 if two_d else ny
    off, ext = P.slab_extent(slab, rank, nranks)
    q = L.Q_OF[stencil]
    dt = torch.float64 if prec == L.LBM_FP64 else torch.float32
    g = torch.full((lay.elements,), -1.0, dtype=dt)
    v = g.view(lay.planes, q, nyy, lay.pitch)
    zz = torch.arange(ext).view(-1, 1, 1, 1) + off
    ii = torch.arange(q).view(1, -1, 1, 1)
    yy = torch.arange(nyy).view(1, 1, -1, 1)
    xx = torch.arange(nx).view(1, 1, 1, -1)
    v[1:ext + 1, :, :, :nx] = fill_value(zz, ii, yy, xx).to(dt)
    return g, lay, off, ext, q, nyy


def _worker(rank, world, port, stencil, prec, shape, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, lay, off, ext, q, nyy = make_grid(stencil, prec, shape, rank, world)
        views = D.HaloViews(g[lay.send_lo:lay.send_lo + lay.halo_elems], g[lay.send_hi:lay.send_hi + lay.halo_elems],
                            g[lay.recv_lo:lay.recv_lo + lay.halo_elems], g[lay.recv_hi:lay.recv_hi + lay.halo_elems])
        D.exchange(views, rank, world)
        out[rank] = g.numpy().copy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("stencil,prec,shape,world", [
    (L.LBM_D3Q27, L.LBM_FP64, (10, 6, 8), 2),
    (L.LBM_D3Q19, L.LBM_FP32, (10, 6, 12), 4),
    (L.LBM_D2Q9, L.LBM_FP64, (12, 8, 1), 2),
])
def test_gloo_halo_exchange(stencil, prec, shape, world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), stencil, prec, shape, out), nprocs=world, join=True)
    xi, opp = P.stencil_info(stencil)
    slab_ax = 1 if stencil == L.LBM_D2Q9 else 2
    nx = shape[0]
    two_d = stencil == L.LBM_D2Q9
    slab = shape[1] if two_d else shape[2]
    for r in range(world):
        g, lay, off, ext, q, nyy = make_grid(stencil, prec, shape, r, world)
        got = np.asarray(out[r]).reshape(lay.planes, q, nyy, lay.pitch)
        up = [i for i in range(q) if xi[i, slab_ax] == 1]
        down = [i for i in range(q) if xi[i, slab_ax] == -1]
        yy = np.arange(nyy).reshape(-1, 1)
        xx = np.arange(nx).reshape(1, -1)
        # bottom ghost: the +1 populations of global plane off - 1 (periodic)
        zlo = (off - 1) % slab
        zhi = (off + ext) % slab
        for i in range(q):
            lo = got[0, i, :, :nx]
            hi = got[ext + 1, i, :, :nx]
            if i in up:
                np.testing.assert_array_equal(lo, fill_value(zlo, i, yy, xx))
            else:
                assert (lo == -1).all()
            if i in down:
                np.testing.assert_array_equal(hi, fill_value(zhi, i, yy, xx))
            else:
                assert (hi == -1).all()
        # interior untouched
        np.testing.assert_array_equal(got[1:ext + 1], g.numpy().reshape(got.shape)[1:ext + 1])


def test_halo_blocks_are_the_crossing_populations():
    """The halo offsets of lbm_grid_layout cover exactly the populations whose slab
    component is +1 (send_hi / recv_lo) or -1 (send_lo / recv_hi)."""
    for st in (L.LBM_D2Q9, L.LBM_D3Q19, L.LBM_D3Q27):
        shape = (16, 8, 1) if st == L.LBM_D2Q9 else (16, 8, 8)
        lay = P.grid_layout(st, L.LBM_FP64, shape, 2)
        xi, _ = P.stencil_info(st)
        ax = 1 if st == L.LBM_D2Q9 else 2
        up = np.flatnonzero(xi[:, ax] == 1)
        down = np.flatnonzero(xi[:, ax] == -1)
        assert lay.halo_elems == len(up) * lay.pop
        assert lay.send_hi % lay.plane == up[0] * lay.pop and lay.send_hi // lay.plane == lay.planes - 2
        assert lay.recv_lo // lay.plane == 0 and lay.recv_lo % lay.plane == up[0] * lay.pop
        assert lay.send_lo // lay.plane == 1 and lay.send_lo % lay.plane == down[0] * lay.pop
        assert lay.recv_hi // lay.plane == lay.planes - 1
        assert list(up) == list(range(up[0], up[0] + len(up)))
        assert list(down) == list(range(down[0], down[0] + len(down)))
        assert lay.pitch % 16 == 0 and lay.pitch >= shape[0]
        # AA (lbm.h): before the odd step the neighbours' boundary slots the odd step reads come
        # in (ghost below: the -1 block, ghost above: the +1 block); after it the ghost-plane
        # writes go back out - the post exchange is the pre exchange with send and recv swapped
        top, bot = lay.planes - 2, 1
        assert (lay.aa_pre_recv_lo // lay.plane, lay.aa_pre_recv_lo % lay.plane) == (0, down[0] * lay.pop)
        assert (lay.aa_pre_recv_hi // lay.plane, lay.aa_pre_recv_hi % lay.plane) == (top + 1, up[0] * lay.pop)
        assert (lay.aa_pre_send_lo // lay.plane, lay.aa_pre_send_lo % lay.plane) == (bot, up[0] * lay.pop)
        assert (lay.aa_pre_send_hi // lay.plane, lay.aa_pre_send_hi % lay.plane) == (top, down[0] * lay.pop)
        assert (lay.aa_post_send_lo, lay.aa_post_send_hi) == (lay.aa_pre_recv_lo, lay.aa_pre_recv_hi)
        assert (lay.aa_post_recv_lo, lay.aa_post_recv_hi) == (lay.aa_pre_send_lo, lay.aa_pre_send_hi)


class _FakePeerLattice:
    """Stands in for a Lattice in PeerRunner's host protocol (no device): records the
    calls and the neighbour infos it was connected with."""

    def __init__(self, rank, nranks):
        self.rank, self.nranks, self.calls = rank, nranks, []

    def peer_export(self):
        info = L.lbm_peer_info()
        info.rank, info.nranks, info.pid = self.rank, self.nranks, os.getpid()
        self.calls.append("export")
        return bytes(info)

    def peer_connect(self, lower, upper):
        lo = L.lbm_peer_info.from_buffer_copy(lower)
        hi = L.lbm_peer_info.from_buffer_copy(upper)
        self.calls.append(("connect", lo.rank, hi.rank))

    def sync(self):
        self.calls.append("sync")

    def peer_prime(self):
        self.calls.append("prime")

    def step(self, n):  # lbm_step on the connected context (the fused push)
        self.calls.append(("step", n))

    def peer_timed_out(self):
        return False


def _peer_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lat = _FakePeerLattice(rank, world)
        runner = D.PeerRunner(lat, rank, world)
        runner.prime()
        runner.step(7)
        runner.check()
        out[rank] = lat.calls
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_peer_runner_host_protocol(world):
    """PeerRunner (the fused-halo driver) on gloo: every rank exports, gathers all infos,
    connects to its periodic lower / upper neighbours, synchronises before the barrier,
    primes, then steps with one library call."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_peer_worker, args=(world, free_port(), out), nprocs=world, join=True)
    for r in range(world):
        calls = out[r]
        lo, hi = (r - 1) % world, (r + 1) % world
        assert calls == ["export", ("connect", lo, hi), "sync", "sync", "prime", ("step", 7)], calls


class _FailingPeerLattice(_FakePeerLattice):
    """Rank `bad` cannot map its neighbours (as without NVLink peer access)."""

    bad = 1

    def peer_connect(self, lower, upper):
        if self.rank == self.bad:
            self.calls.append("connect-failed")
            raise L.LbmError(L.LBM_ECUDA, "cudaIpcOpenMemHandle: peer access unsupported")
        super().peer_connect(lower, upper)

    def peer_disconnect(self):
        self.calls.append("disconnect")


def _peer_fail_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lat = _FailingPeerLattice(rank, world)
        try:
            D.PeerRunner(lat, rank, world)
            out[rank] = ("no error", lat.calls)
        except D.PeerUnavailable as ex:
            out[rank] = (str(ex), lat.calls)
        dist.barrier()  # the group is still usable: the fallback's collectives line up
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_peer_runner_fails_collectively(world):
    """One rank's failed peer mapping makes EVERY rank raise PeerUnavailable (no deadlock, no
    rank left on the fused path); ranks that had connected unmap their neighbours again, so
    bench.py's fallback to the NCCL exchange is taken by the whole group."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_peer_fail_worker, args=(world, free_port(), out), nprocs=world, join=True)
    for r in range(world):
        msg, calls = out[r]
        assert "unavailable on ranks [1]" in msg, msg
        if r == _FailingPeerLattice.bad:
            assert calls == ["export", "connect-failed"], calls
        else:
            assert calls[-1] == "disconnect" and calls[0] == "export", calls
