"""Thin ctypes binding of include/lbm.h (argument marshalling only).

Every step of the hot path runs in liblbm.so's CUDA kernels; this module only
converts numpy arrays to pointers and status codes to exceptions.  There is
no CPU fallback: if liblbm.so cannot be loaded, importing the binding raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblbm.so")

# enums of include/lbm.h
LBM_OK, LBM_EINVAL, LBM_EUNSUPPORTED, LBM_ENOMEM, LBM_ECUDA, LBM_ENCCL, LBM_ENUMERIC = 0, -1, -2, -3, -4, -5, -6
LBM_D2Q9, LBM_D3Q19, LBM_D3Q27 = 0, 1, 2
LBM_SPACE_POPULATION, LBM_SPACE_RAW, LBM_SPACE_CENTRAL, LBM_SPACE_CUMULANT, LBM_SPACE_RAW_WO = 0, 1, 2, 3, 4
(LBM_EQ_ABSOLUTE, LBM_EQ_DELTA, LBM_EQ_SWE, LBM_EQ_DISCRETE, LBM_EQ_DISCRETE_DELTA,
 LBM_EQ_ABSOLUTE_F0) = 0, 1, 2, 3, 4, 5
LBM_FP64, LBM_FP32 = 0, 1
LBM_PULL, LBM_AA, LBM_ESOTERIC_PULL, LBM_ESOTERIC_TWIST, LBM_ESOTERIC_PUSH = 0, 1, 2, 3, 4
LBM_BC_PERIODIC, LBM_BC_NOSLIP = 0, 1
LBM_FORCE_GUO, LBM_FORCE_HE = 0, 1
LBM_REGION_ALL, LBM_REGION_BOUNDARY, LBM_REGION_INTERIOR = 0, 1, 2
LBM_REGION_PAIR_INTERIOR, LBM_REGION_PAIR_BOUNDARY1, LBM_REGION_PAIR_BOUNDARY2 = 3, 4, 5
LBM_REGION_TRIPLE_INTERIOR, LBM_REGION_TRIPLE_BOUNDARY1, LBM_REGION_TRIPLE_BOUNDARY2, LBM_REGION_TRIPLE_BOUNDARY3 = \
    6, 7, 8, 9

Q_OF = {LBM_D2Q9: 9, LBM_D3Q19: 19, LBM_D3Q27: 27}

STATUS_NAMES = {0: "LBM_OK", -1: "LBM_EINVAL", -2: "LBM_EUNSUPPORTED", -3: "LBM_ENOMEM", -4: "LBM_ECUDA",
                -5: "LBM_ENCCL", -6: "LBM_ENUMERIC"}


class LbmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


DEV_ALLOC = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
DEV_FREE = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class lbm_domain(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("bc", (ctypes.c_int * 2) * 3), ("precision", ctypes.c_int), ("streaming", ctypes.c_int),
                ("swe_g", ctypes.c_double), ("device", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("nccl_id", ctypes.c_void_p),
                ("dev_alloc", DEV_ALLOC), ("dev_free", DEV_FREE), ("alloc_user", ctypes.c_void_p)]


class lbm_halo(ctypes.Structure):
    _fields_ = [("send_lo", ctypes.c_void_p), ("send_hi", ctypes.c_void_p), ("recv_lo", ctypes.c_void_p),
                ("recv_hi", ctypes.c_void_p), ("bytes", ctypes.c_size_t)]


class lbm_layout(ctypes.Structure):
    _fields_ = [(n, ctypes.c_size_t) for n in (
        "pitch", "pop", "plane", "planes", "elements", "send_lo", "send_hi", "recv_lo", "recv_hi", "halo_elems",
        "aa_pre_send_lo", "aa_pre_send_hi", "aa_pre_recv_lo", "aa_pre_recv_hi",
        "aa_post_send_lo", "aa_post_send_hi", "aa_post_recv_lo", "aa_post_recv_hi")]


class lbm_diagnostics(ctypes.Structure):
    _fields_ = [("mass", ctypes.c_double), ("momentum", ctypes.c_double * 3), ("kinetic_energy", ctypes.c_double)]


class lbm_info(ctypes.Structure):
    _fields_ = [("q", ctypes.c_int), ("d", ctypes.c_int), ("offset", ctypes.c_int), ("extent", ctypes.c_int),
                ("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int), ("pitch", ctypes.c_size_t),
                ("bytes_per_element", ctypes.c_size_t), ("device_bytes", ctypes.c_size_t),
                ("steps_done", ctypes.c_longlong), ("rate_specialization", ctypes.c_int),
                ("temporal_blocking", ctypes.c_int), ("cuda_graph_steps", ctypes.c_int),
                ("resident_cluster", ctypes.c_int), ("peer_wait_host", ctypes.c_int)]


class lbm_peer_info(ctypes.Structure):
    _fields_ = [("grid_ipc", (ctypes.c_ubyte * 64) * 2), ("flags_ipc", ctypes.c_ubyte * 64),
                ("grid", ctypes.c_void_p * 2), ("flags", ctypes.c_void_p), ("pid", ctypes.c_longlong),
                ("device", ctypes.c_int), ("rank", ctypes.c_int), ("nranks", ctypes.c_int),
                ("stencil", ctypes.c_int), ("precision", ctypes.c_int), ("nx", ctypes.c_int),
                ("ny", ctypes.c_int), ("nz", ctypes.c_int), ("grid_off", ctypes.c_longlong * 2),
                ("uuid", ctypes.c_ubyte * 16)]


_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p

# (name, restype, argtypes) for every symbol of include/lbm.h
SIGNATURES = [
    ("lbm_create", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_int,
                                  ctypes.POINTER(lbm_domain), ctypes.c_int, ctypes.POINTER(_vp)]),
    ("lbm_destroy", ctypes.c_int, [_vp]),
    ("lbm_last_error", ctypes.c_char_p, [_vp]),
    ("lbm_get_info", ctypes.c_int, [_vp, ctypes.POINTER(lbm_info)]),
    ("lbm_init_macroscopic", ctypes.c_int, [_vp, _dp, _dp]),
    ("lbm_step", ctypes.c_int, [_vp, ctypes.c_int]),
    ("lbm_nccl_get_unique_id", ctypes.c_int, [_vp]),
    ("lbm_step_region", ctypes.c_int, [_vp, ctypes.c_int, _vp]),
    ("lbm_swap", ctypes.c_int, [_vp]),
    ("lbm_get_halo", ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(lbm_halo)]),
    ("lbm_sync", ctypes.c_int, [_vp]),
    ("lbm_peer_export", ctypes.c_int, [_vp, ctypes.POINTER(lbm_peer_info)]),
    ("lbm_peer_connect", ctypes.c_int, [_vp, ctypes.POINTER(lbm_peer_info), ctypes.POINTER(lbm_peer_info)]),
    ("lbm_peer_prime", ctypes.c_int, [_vp]),
    ("lbm_step_peer", ctypes.c_int, [_vp, ctypes.c_int]),
    ("lbm_peer_status", ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int)]),
    ("lbm_get_macroscopic", ctypes.c_int, [_vp, _dp, _dp]),
    ("lbm_get_populations", ctypes.c_int, [_vp, _dp]),
    ("lbm_set_populations", ctypes.c_int, [_vp, _dp]),
    ("lbm_set_steps", ctypes.c_int, [_vp, ctypes.c_longlong]),
    ("lbm_get_cells", ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_longlong), ctypes.c_longlong, _dp]),
    ("lbm_get_diagnostics", ctypes.c_int, [_vp, ctypes.POINTER(lbm_diagnostics)]),
    ("lbm_set_force", ctypes.c_int, [_vp, _dp]),
    ("lbm_set_force_model", ctypes.c_int, [_vp, ctypes.c_int]),
    ("lbm_check_finite", ctypes.c_int, [_vp]),
    ("lbm_test_collide", ctypes.c_int, [_vp, _dp, _dp, ctypes.c_longlong]),
    ("lbm_stencil_info", ctypes.c_int, [ctypes.c_int, _ip, _ip, _ip]),
    ("lbm_slab_extent", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _ip, _ip]),
    ("lbm_version", ctypes.c_char_p, []),
    ("lbm_grid_layout", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.POINTER(lbm_layout)]),
    ("lbm_kernel_attributes", ctypes.c_int, [_vp, _ip, _ip]),
    ("lbm_device_grid", ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_size_t)]),
    ("lbm_stream", _vp, [_vp]),
]

_lib = None


def lib():
    """The loaded liblbm.so.  Raises if the CUDA library is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run paper_2211_02435_b200.build.build() "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def _check(status: int, ctx=None):
    if status != LBM_OK:
        msg = lib().lbm_last_error(ctx)
        raise LbmError(status, msg.decode() if msg else "")


def stencil_info(stencil: int):
    q = ctypes.c_int()
    xi = np.zeros(27 * 3, np.int32)
    opp = np.zeros(27, np.int32)
    _check(lib().lbm_stencil_info(stencil, ctypes.byref(q), xi.ctypes.data_as(_ip), opp.ctypes.data_as(_ip)))
    n = q.value
    return xi[: 3 * n].reshape(n, 3).copy(), opp[:n].copy()


def slab_extent(extent: int, rank: int, nranks: int):
    off, ext = ctypes.c_int(), ctypes.c_int()
    _check(lib().lbm_slab_extent(extent, rank, nranks, ctypes.byref(off), ctypes.byref(ext)))
    return off.value, ext.value


def grid_layout(stencil: int, precision: int, shape, nranks: int = 1) -> lbm_layout:
    """Host-only: the device grid layout of a rank's slab (element offsets)."""
    out = lbm_layout()
    nx, ny, nz = shape
    _check(lib().lbm_grid_layout(int(stencil), int(precision), int(nx), int(ny), int(nz), int(nranks),
                                 ctypes.byref(out)))
    return out


def version() -> str:
    return lib().lbm_version().decode()


def nccl_get_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0; pass it to every rank's Lattice(nccl_id=...))."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().lbm_nccl_get_unique_id(buf))
    return buf.raw


class Lattice:
    """One lbm_ctx: a rank's slab of an MRT LBM simulation on a CUDA device.

    Arguments mirror lbm_create(); shape = (nx, ny, nz) global (2D: nz = 1);
    bc = [[x_lo, x_hi], [y_lo, y_hi], [z_lo, z_hi]] of LBM_BC_*.
    """

    def __init__(self, stencil, space, equilibrium, rates, shape, zero_centered=True, precision=LBM_FP64,
                 streaming=LBM_PULL, bc=None, swe_g=0.0, device=0, stream=None, rank=0, nranks=1, nccl_id=None,
                 allocator=None):
        """nccl_id: 128 bytes from nccl_get_unique_id() (same on every rank): in-library NCCL halo
        exchange in lbm_step (collective create).  allocator: optional (alloc(nbytes) -> int device
        pointer, free(ptr)) pair used for the population grids (lbm_domain.dev_alloc/dev_free)."""
        L = lib()
        dom = lbm_domain()
        dom.nx, dom.ny, dom.nz = (int(v) for v in shape)
        bc = bc if bc is not None else [[LBM_BC_PERIODIC] * 2] * 3
        for a in range(3):
            for s in range(2):
                dom.bc[a][s] = int(bc[a][s])
        dom.precision = int(precision)
        dom.streaming = int(streaming)
        dom.swe_g = float(swe_g)
        dom.device = int(device)
        dom.stream = stream
        dom.rank = int(rank)
        dom.nranks = int(nranks)
        self._nccl_id = None
        if nccl_id is not None:
            assert len(nccl_id) == 128, "an ncclUniqueId is 128 bytes"
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            dom.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        self._alloc_cbs = None
        if allocator is not None:
            alloc_fn, free_fn = allocator
            self._alloc_cbs = (DEV_ALLOC(lambda n, _u: int(alloc_fn(int(n))) or None),
                               DEV_FREE(lambda p, _u: free_fn(int(p))))
            dom.dev_alloc, dom.dev_free = self._alloc_cbs
        r = np.ascontiguousarray(np.asarray(rates, dtype=np.float64).reshape(-1))
        h = _vp()
        self._ctx = None
        _check(L.lbm_create(int(stencil), int(space), int(equilibrium), _d(r), r.size, ctypes.byref(dom),
                            1 if zero_centered else 0, ctypes.byref(h)))
        self._ctx = h
        self.stencil, self.space, self.equilibrium = int(stencil), int(space), int(equilibrium)
        self.zero_centered = bool(zero_centered)
        self.precision, self.streaming = int(precision), int(streaming)
        info = self.info()
        self.q, self.d = info.q, info.d
        self.global_shape = (info.nx, info.ny, info.nz)
        self.offset, self.extent = info.offset, info.extent
        nx, ny, nz = self.global_shape
        # host array shape of this rank's slab: [z][y][x] (2D: [1][y_local][x])
        self.local_shape = (1, self.extent, nx) if self.d == 2 else (self.extent, ny, nx)

    # -- lifecycle
    def close(self):
        if self._ctx:
            lib().lbm_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- C ABI, same names
    def info(self) -> lbm_info:
        i = lbm_info()
        _check(lib().lbm_get_info(self._ctx, ctypes.byref(i)), self._ctx)
        return i

    @property
    def cells(self) -> int:
        z, y, x = self.local_shape
        return z * y * x

    def init_macroscopic(self, rho, u):
        rho = np.ascontiguousarray(rho, dtype=np.float64).reshape(-1)
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        assert rho.size == self.cells and u.size == self.d * self.cells
        _check(lib().lbm_init_macroscopic(self._ctx, _d(rho), _d(u)), self._ctx)

    def step(self, n=1):
        _check(lib().lbm_step(self._ctx, int(n)), self._ctx)

    def step_region(self, region, stream=None):
        _check(lib().lbm_step_region(self._ctx, int(region), stream), self._ctx)

    def swap(self):
        _check(lib().lbm_swap(self._ctx), self._ctx)

    def get_halo(self, which=0) -> lbm_halo:
        h = lbm_halo()
        _check(lib().lbm_get_halo(self._ctx, int(which), ctypes.byref(h)), self._ctx)
        return h

    def sync(self):
        _check(lib().lbm_sync(self._ctx), self._ctx)

    # fused halo push between slab contexts (include/lbm.h lbm_peer_*)
    def peer_export(self) -> bytes:
        info = lbm_peer_info()
        _check(lib().lbm_peer_export(self._ctx, ctypes.byref(info)), self._ctx)
        return bytes(info)

    def peer_connect(self, lower: bytes, upper: bytes):
        lo = lbm_peer_info.from_buffer_copy(lower)
        hi = lbm_peer_info.from_buffer_copy(upper)
        _check(lib().lbm_peer_connect(self._ctx, ctypes.byref(lo), ctypes.byref(hi)), self._ctx)

    def peer_disconnect(self):
        _check(lib().lbm_peer_connect(self._ctx, None, None), self._ctx)

    def peer_prime(self):
        _check(lib().lbm_peer_prime(self._ctx), self._ctx)

    def step_peer(self, n=1):
        _check(lib().lbm_step_peer(self._ctx, int(n)), self._ctx)

    def peer_timed_out(self) -> bool:
        v = ctypes.c_int(0)
        _check(lib().lbm_peer_status(self._ctx, ctypes.byref(v)), self._ctx)
        return bool(v.value)

    def get_macroscopic(self, out=None):
        z, y, x = self.local_shape
        rho = np.empty((z, y, x)) if out is None else out[0]
        u = np.empty((self.d, z, y, x)) if out is None else out[1]
        _check(lib().lbm_get_macroscopic(self._ctx, _d(rho), _d(u)), self._ctx)
        return rho, u

    def get_populations(self):
        f = np.empty((self.q,) + self.local_shape)
        _check(lib().lbm_get_populations(self._ctx, _d(f)), self._ctx)
        return f

    def set_force(self, force, model=None):
        """Uniform body force density (include/lbm.h lbm_set_force); model: LBM_FORCE_GUO or
        LBM_FORCE_HE (lbm_set_force_model), None keeps the current one (default Guo)."""
        if model is not None:
            _check(lib().lbm_set_force_model(self._ctx, int(model)), self._ctx)
        F = np.ascontiguousarray(np.asarray(force, dtype=np.float64).reshape(-1))
        F = np.concatenate([F, np.zeros(3 - F.size)]) if F.size < 3 else F
        _check(lib().lbm_set_force(self._ctx, _d(np.ascontiguousarray(F))), self._ctx)

    def get_diagnostics(self):
        """dict(mass, momentum[3], kinetic_energy) of this slab (device sums, fp64)."""
        d = lbm_diagnostics()
        _check(lib().lbm_get_diagnostics(self._ctx, ctypes.byref(d)), self._ctx)
        return {"mass": d.mass, "momentum": list(d.momentum), "kinetic_energy": d.kinetic_energy}

    def get_cells(self, cells):
        """Canonical populations [n][q] of local linear cell indices x + nx (y + ny z)."""
        idx = np.ascontiguousarray(np.asarray(cells, dtype=np.int64).reshape(-1))
        out = np.empty((idx.size, self.q))
        _check(lib().lbm_get_cells(self._ctx, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), idx.size,
                                   _d(out)), self._ctx)
        return out

    def set_populations(self, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        assert f.size == self.q * self.cells
        _check(lib().lbm_set_populations(self._ctx, _d(f)), self._ctx)

    def check_finite(self):
        _check(lib().lbm_check_finite(self._ctx), self._ctx)

    def run(self, n, check_every=0, callback=None, every=0):
        """n steps; optionally lbm_check_finite every `check_every` steps (raises LbmError
        LBM_ENUMERIC with the step index) and callback(self, steps_done) every `every` steps.
        Intervals count from the start of this call; chunks end on every multiple of either."""
        done = 0
        while done < n:
            k = n - done
            if check_every > 0:
                k = min(k, check_every - done % check_every)
            if every > 0:
                k = min(k, every - done % every)
            self.step(k)
            done += k
            if check_every > 0 and done % check_every == 0:
                self.check_finite()
            if callback is not None and every > 0 and done % every == 0:
                callback(self, self.info().steps_done)

    # -- checkpoint / restart: the canonical state (independent of the streaming pattern)
    def save(self, path, rates=None):
        """Checkpoint of this rank's slab: canonical populations + method metadata (npz)."""
        info = self.info()
        np.savez(path, f=self.get_populations(), steps=info.steps_done, stencil=self.stencil, space=self.space,
                 equilibrium=self.equilibrium, zero_centered=self.zero_centered, shape=np.array(self.global_shape),
                 offset=self.offset, extent=self.extent, precision=self.precision, streaming=self.streaming,
                 rates=np.asarray(rates if rates is not None else [], dtype=np.float64))

    def load(self, path, rates=None):
        """Restore a checkpoint written by save() for the same method, precision and slab.
        Returns the saved step count and restores the context's counter (lbm_info.steps_done,
        lbm_set_steps) to it; the canonical state is independent of the counter.  On
        several ranks the next lbm_step exchanges the halo first (an external-exchange driver,
        SlabRunner, must call prime())."""
        d = np.load(path)
        for k, v in (("stencil", self.stencil), ("space", self.space), ("equilibrium", self.equilibrium),
                     ("zero_centered", self.zero_centered), ("offset", self.offset), ("extent", self.extent),
                     ("precision", self.precision)):
            if k in d and int(d[k]) != int(v):
                raise ValueError(f"checkpoint {k} = {d[k]} does not match this lattice ({v})")
        if tuple(d["shape"]) != tuple(self.global_shape):
            raise ValueError("checkpoint lattice shape differs")
        if rates is not None and "rates" in d and d["rates"].size and not np.array_equal(
                d["rates"], np.asarray(rates, dtype=np.float64).reshape(-1)):
            raise ValueError("checkpoint relaxation rates differ")
        self.set_populations(d["f"])
        _check(lib().lbm_set_steps(self._ctx, int(d["steps"])), self._ctx)
        return int(d["steps"])

    def test_collide(self, f_in):
        f_in = np.ascontiguousarray(f_in, dtype=np.float64)
        assert f_in.ndim == 2 and f_in.shape[1] == self.q
        out = np.empty_like(f_in)
        _check(lib().lbm_test_collide(self._ctx, _d(f_in), _d(out), f_in.shape[0]), self._ctx)
        return out

    def kernel_attributes(self):
        r, l = ctypes.c_int(), ctypes.c_int()
        _check(lib().lbm_kernel_attributes(self._ctx, ctypes.byref(r), ctypes.byref(l)), self._ctx)
        return r.value, l.value

    def device_grid(self, which=0):
        p, b = _vp(), ctypes.c_size_t()
        _check(lib().lbm_device_grid(self._ctx, int(which), ctypes.byref(p), ctypes.byref(b)), self._ctx)
        return p.value, b.value

    @property
    def stream(self):
        return lib().lbm_stream(self._ctx)
