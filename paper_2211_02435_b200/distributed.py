"""Multi-rank slab decomposition driver (one process per GPU).

The lattice is cut into slabs along its slab axis (z in 3D, y in 2D), one per
rank.  Pull streaming couples a slab to its neighbours only
through one ghost plane per face, so one halo exchange per time step suffices:
after the two boundary planes of the next grid are computed, each rank sends
its top plane's slab-component +1 population block up and its bottom plane's
-1 block down, while the interior planes are updated concurrently.  Thanks to
the population ordering of include/lbm.h each block is contiguous in memory,
so the exchange is zero-copy.

Transport is torch.distributed point-to-point (NCCL over NVLink on GPUs, gloo
on CPU for tests); `LocalTransport` connects several contexts of one process
(used by the single-GPU equivalence tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import lbm as L

TAG_UP, TAG_DOWN = 11, 12


def neighbours(rank: int, nranks: int):
    """(lower, upper) neighbour ranks with periodic wrap along the slab axis."""
    return (rank - 1) % nranks, (rank + 1) % nranks


@dataclass
class HaloViews:
    send_lo: object
    send_hi: object
    recv_lo: object
    recv_hi: object


def exchange(views: HaloViews, rank: int, nranks: int, group=None):
    """One halo exchange with torch.distributed P2P.  send_hi -> upper's recv_lo
    (tag UP), send_lo -> lower's recv_hi (tag DOWN).  Works on CUDA tensors
    (NCCL) and CPU tensors (gloo).  Returns after completion."""
    import torch.distributed as dist

    lo, hi = neighbours(rank, nranks)
    ops = [
        dist.P2POp(dist.isend, views.send_hi, hi, group, TAG_UP),
        dist.P2POp(dist.isend, views.send_lo, lo, group, TAG_DOWN),
        dist.P2POp(dist.irecv, views.recv_lo, lo, group, TAG_UP),
        dist.P2POp(dist.irecv, views.recv_hi, hi, group, TAG_DOWN),
    ]
    for r in dist.batch_isend_irecv(ops):
        r.wait()


class _CudaArray:
    """Minimal __cuda_array_interface__ wrapper to view library memory from torch."""

    def __init__(self, ptr: int, nelem: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (nelem,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def halo_views(lat: "L.Lattice", which: int) -> HaloViews:
    """torch CUDA tensors aliasing the halo blocks of a context's grid."""
    import torch

    h = lat.get_halo(which)
    esize = 8 if lat.precision == L.LBM_FP64 else 4
    typestr = "<f8" if esize == 8 else "<f4"
    n = h.bytes // esize
    dev = torch.device("cuda", torch.cuda.current_device())
    mk = lambda p: torch.as_tensor(_CudaArray(p, n, typestr), device=dev)
    return HaloViews(mk(h.send_lo), mk(h.send_hi), mk(h.recv_lo), mk(h.recv_hi))


class TorchTransport:
    """Halo exchange between the processes of a torch.distributed group.

    NCCL moves the device blocks directly (zero-copy, NVLink).  A gloo group (CPU
    transport: tests, or several ranks sharing one GPU) stages the blocks through
    pinned host buffers."""

    def __init__(self, lat: "L.Lattice", rank: int, nranks: int, group=None):
        import torch.distributed as dist

        self.lat, self.rank, self.nranks, self.group = lat, rank, nranks, group
        self.staged = dist.get_backend(group) == "gloo"
        # halo views of both grids (they alternate every step)
        self._views = {}
        self._host = None

    def _get(self, which):
        key = (which, self.lat.get_halo(which).send_lo)
        if key not in self._views:
            self._views[key] = halo_views(self.lat, which)
        return self._views[key]

    def exchange(self, which: int):
        v = self._get(which)
        if not self.staged:
            exchange(v, self.rank, self.nranks, self.group)
            return
        import torch

        if self._host is None:
            mk = lambda t: torch.empty(t.shape, dtype=t.dtype).pin_memory()
            self._host = HaloViews(mk(v.send_lo), mk(v.send_hi), mk(v.recv_lo), mk(v.recv_hi))
        h = self._host
        h.send_lo.copy_(v.send_lo)  # synchronous D2H: waits for the boundary planes
        h.send_hi.copy_(v.send_hi)
        exchange(h, self.rank, self.nranks, self.group)
        v.recv_lo.copy_(h.recv_lo, non_blocking=True)
        v.recv_hi.copy_(h.recv_hi, non_blocking=True)


class LocalTransport:
    """Connects the slab contexts of ONE process (ranks 0..n-1 on one device)."""

    def __init__(self, lats):
        self.lats = list(lats)

    def exchange_all(self, which: int):
        import torch

        n = len(self.lats)
        views = [halo_views(l, which) for l in self.lats]
        torch.cuda.synchronize()
        for r in range(n):
            lo, hi = neighbours(r, n)
            views[hi].recv_lo.copy_(views[r].send_hi)
            views[lo].recv_hi.copy_(views[r].send_lo)
        torch.cuda.synchronize()


def exchange_after_boundary(lat: "L.Lattice") -> int:
    """Which halo (lbm_get_halo) to exchange once the boundary planes of this step are done:
    pull: the next grid (1).  AA (lbm.h): after an odd step the ghost-plane writes return
    to the neighbours ("post", 1); after an even step the boundary slots the next odd step
    reads go out ("pre", 0)."""
    if lat.streaming == L.LBM_PULL:
        return 1
    odd = lat.info().steps_done % 2 == 0  # state A -> this step runs the odd kernel
    return 1 if odd else 0


def supports_pairs(lat: "L.Lattice") -> bool:
    """The context runs two-step sweeps across ranks (LBM_REGION_PAIR_*, lbm_get_halo(2))."""
    try:
        lat.get_halo(2)
        return True
    except L.LbmError:
        return False


def supports_triples(lat: "L.Lattice") -> bool:
    """The context runs three-step sweeps across ranks (LBM_REGION_TRIPLE_*, lbm_get_halo(3/4):
    2D slabs of >= 10 rows)."""
    try:
        lat.get_halo(3)
        return True
    except L.LbmError:
        return False


def step_local(lats, n: int, pairs: bool = False):
    """n time steps of all slab contexts of one process (LocalTransport), with the
    same boundary/interior split as the multi-process driver (pairs: the fused-step regions,
    triples where every context has them, then pairs)."""
    tr = LocalTransport(lats)
    if pairs and all(supports_triples(l) for l in lats):
        while n >= 3:
            for l in lats:
                l.step_region(L.LBM_REGION_TRIPLE_INTERIOR)
                l.step_region(L.LBM_REGION_TRIPLE_BOUNDARY1)
            for l in lats:
                l.sync()
            tr.exchange_all(3)
            for l in lats:
                l.step_region(L.LBM_REGION_TRIPLE_BOUNDARY2)
            for l in lats:
                l.sync()
            tr.exchange_all(4)
            for l in lats:
                l.step_region(L.LBM_REGION_TRIPLE_BOUNDARY3)
            for l in lats:
                l.sync()
            tr.exchange_all(1)
            for l in lats:
                l.swap()
            n -= 3
    if pairs and all(supports_pairs(l) for l in lats):
        while n >= 2:
            for l in lats:
                l.step_region(L.LBM_REGION_PAIR_INTERIOR)
                l.step_region(L.LBM_REGION_PAIR_BOUNDARY1)
            for l in lats:
                l.sync()
            tr.exchange_all(2)
            for l in lats:
                l.step_region(L.LBM_REGION_PAIR_BOUNDARY2)
            for l in lats:
                l.sync()
            tr.exchange_all(1)
            for l in lats:
                l.swap()
            n -= 2
    for _ in range(n):
        which = exchange_after_boundary(lats[0])
        for l in lats:
            l.step_region(L.LBM_REGION_BOUNDARY)
        for l in lats:
            l.sync()
        tr.exchange_all(which)
        for l in lats:
            l.step_region(L.LBM_REGION_INTERIOR)
        for l in lats:
            l.sync()
            l.swap()


def prime_local(lats):
    """Fill the ghost planes after init/set (pull: current grid; AA: the pre-odd halo)."""
    LocalTransport(lats).exchange_all(0)


class SlabRunner:
    """Multi-process time stepping of one rank's slab: boundary planes, then the
    halo exchange (NCCL P2P on its own stream) overlapped with the interior planes."""

    def __init__(self, lat: "L.Lattice", rank: int, nranks: int, group=None, pairs=None):
        """pairs: None = two-step sweeps across ranks where the context supports them (equal to
        the single-rank run to rounding), False = single steps (bitwise equal to it), True =
        require them (ValueError if unsupported).  The choice must be the same on every rank."""
        import torch

        self.lat, self.rank, self.nranks = lat, rank, nranks
        self.tr = TorchTransport(lat, rank, nranks, group)
        self.s_int = torch.cuda.Stream()
        self.s_main = torch.cuda.current_stream()
        can = lat.streaming == L.LBM_PULL and supports_pairs(lat)
        if pairs and not can:
            raise ValueError("this context has no two-step regions (LBM_REGION_PAIR_*)")
        self.pairs = can if pairs is None else bool(pairs)
        self.triples = self.pairs and supports_triples(lat)  # 2D slabs of >= 10 rows

    def prime(self):
        self.lat.sync()
        self.tr.exchange(0)

    def step(self, n: int = 1):
        import torch

        main = self.s_main
        # three fused steps per triple (2D): the interior sweep on s_int overlaps the three
        # boundary steps and their exchanges (level-1 / level-2 scratch rows, next-grid halo)
        while self.triples and n >= 3:
            ev = torch.cuda.Event()
            ev.record(main)
            self.s_int.wait_event(ev)
            self.lat.step_region(L.LBM_REGION_TRIPLE_INTERIOR, self.s_int.cuda_stream)
            for region, which in ((L.LBM_REGION_TRIPLE_BOUNDARY1, 3), (L.LBM_REGION_TRIPLE_BOUNDARY2, 4),
                                  (L.LBM_REGION_TRIPLE_BOUNDARY3, 1)):
                self.lat.step_region(region, main.cuda_stream)
                with torch.cuda.stream(main):
                    self.tr.exchange(which)
            main.wait_stream(self.s_int)
            self.lat.swap()
            n -= 3
        # two fused steps per pair: the interior sweep on s_int overlaps both boundary steps and
        # both exchanges (scratch halo after the first, next-grid halo after the second)
        while self.pairs and n >= 2:
            ev = torch.cuda.Event()
            ev.record(main)
            self.s_int.wait_event(ev)
            self.lat.step_region(L.LBM_REGION_PAIR_INTERIOR, self.s_int.cuda_stream)
            self.lat.step_region(L.LBM_REGION_PAIR_BOUNDARY1, main.cuda_stream)
            with torch.cuda.stream(main):
                self.tr.exchange(2)
            self.lat.step_region(L.LBM_REGION_PAIR_BOUNDARY2, main.cuda_stream)
            with torch.cuda.stream(main):
                self.tr.exchange(1)
            main.wait_stream(self.s_int)
            self.lat.swap()
            n -= 2
        for _ in range(n):
            which = exchange_after_boundary(self.lat)
            # boundary planes on the main stream, then the exchange (NCCL waits on main)
            self.lat.step_region(L.LBM_REGION_BOUNDARY, main.cuda_stream)
            ev = torch.cuda.Event()
            ev.record(main)
            self.s_int.wait_event(ev)
            self.lat.step_region(L.LBM_REGION_INTERIOR, self.s_int.cuda_stream)
            with torch.cuda.stream(main):
                self.tr.exchange(which)
            main.wait_stream(self.s_int)
            self.lat.swap()


def connect_local(lats):
    """Fused halo push (lbm_peer_*) between the slab contexts of ONE process: plain device
    pointers instead of CUDA IPC.  Call step_peer_local afterwards."""
    infos = [l.peer_export() for l in lats]
    n = len(lats)
    for r, l in enumerate(lats):
        lo, hi = neighbours(r, n)
        l.peer_connect(infos[lo], infos[hi])
    for l in lats:
        l.sync()
    for l in lats:
        l.peer_prime()


def on_ranks(lats, fn):
    """fn(lat) for every context of one process, concurrently from one host thread each (the
    ctypes calls release the GIL).  Contexts whose neighbours share their GPU order the peer
    phases on the host (lbm_peer_connect): a context's lbm_step blocks until its neighbours
    enqueued and completed their previous phase, so each needs its own thread."""
    import threading

    errs = [None] * len(lats)

    def run(k):
        try:
            fn(lats[k])
        except BaseException as ex:  # noqa: BLE001 — re-raised below
            errs[k] = ex

    ts = [threading.Thread(target=run, args=(k,)) for k in range(len(lats))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e


def step_peer_local(lats, n: int, chunk: int = 1):
    """n steps of every context of one process with the fused halo push (lbm_step on the
    connected contexts).  Host-ordered contexts (neighbours on the same GPU, the only case on
    a one-GPU box) run in one host thread each; device-ordered ones (every neighbour on another
    GPU) are enqueued from this thread, interleaved in chunks of `chunk` steps (a context waits
    on the GPU for its neighbours; chunk = 2 lets the two-step sweeps run across ranks)."""
    if any(l.info().peer_wait_host for l in lats):
        def run(l):
            done = 0
            while done < n:
                k = min(chunk, n - done)
                l.step(k)
                done += k
        on_ranks(lats, run)
    else:
        done = 0
        while done < n:
            k = min(chunk, n - done)
            for l in lats:
                l.step(k)
            done += k
    for l in lats:
        l.sync()
        assert not l.peer_timed_out(), "a neighbour wait timed out"


class PeerUnavailable(RuntimeError):
    """Raised on EVERY rank when any rank cannot set up the fused halo push."""


class PeerRunner:
    """Multi-process time stepping with the fused halo push: the boundary-plane kernel
    stores the slab-crossing populations straight into the neighbours' ghost planes
    (NVLink peer memory through CUDA IPC; include/lbm.h lbm_peer_*), device-side
    completion flags replace the per-step exchange call.  The host transport of the
    torch.distributed group only carries the one-time handle exchange and barriers."""

    def __init__(self, lat: "L.Lattice", rank: int, nranks: int, group=None):
        import torch.distributed as dist

        self.lat, self.rank, self.nranks, self.group = lat, rank, nranks, group
        # collective setup: every rank takes part in every gather even when its own export or
        # connect fails, and either all ranks run the fused push or none does (a rank that
        # mapped its neighbours unmaps them again), so a fallback cannot deadlock the group
        err = None
        try:
            mine = lat.peer_export()
        except Exception as ex:  # noqa: BLE001 — reported collectively below
            mine, err = None, ex
        infos = [None] * nranks
        dist.all_gather_object(infos, mine, group=group)
        lo, hi = neighbours(rank, nranks)
        connected = False
        if err is None and infos[lo] is not None and infos[hi] is not None:
            try:
                lat.peer_connect(infos[lo], infos[hi])
                lat.sync()
                connected = True
            except Exception as ex:  # noqa: BLE001
                err = ex
        oks = [None] * nranks
        dist.all_gather_object(oks, connected, group=group)
        if not all(oks):
            if connected:
                lat.peer_disconnect()
            bad = [r for r, o in enumerate(oks) if not o]
            raise PeerUnavailable(f"rank {rank}: fused halo push unavailable on ranks {bad}"
                                  + (f" ({err})" if err else ""))
        dist.barrier(group=group)

    def prime(self):
        import torch.distributed as dist

        self.lat.sync()
        dist.barrier(group=self.group)
        self.lat.peer_prime()

    def step(self, n: int = 1):
        self.lat.step(n)  # lbm_step runs the fused push on a connected context (collective)

    def check(self):
        if self.lat.peer_timed_out():
            raise RuntimeError(f"rank {self.rank}: a wait for a neighbour's halo timed out")


def gather_slabs(local_arrays, axis: int):
    """Concatenate per-rank host arrays along the slab axis (helper for tests)."""
    return np.concatenate(local_arrays, axis=axis)
