#!/usr/bin/env python
"""bench.py — throughput of the fused MRT stream–collide hot path on B200.

Default workload (BASELINE.json metric "MLUPS (D3Q27 cumulant fp64) at 1/2/4/8
B200; % of HBM roofline", config 4): D3Q27 cumulant LBM, fp64, zero-centered
storage relaxed against the absolute equilibrium, two-grid pull streaming,
Taylor-Green vortex (eq:TGA_init, u0 = 0.05) on a z-slab-decomposed periodic box
of 1024 x 1024 x (128 N) cells, N = number of GPUs (weak scaling: N = 8 is the
1024^3 box).  One "step" is one time step of the whole lattice.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c3|c2_f64|c2_f32|c1|c5]
  python bench.py --impl reference ...   # the CPU oracle on the host cores

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

BASELINE_METRIC = "MLUPS (D3Q27 cumulant fp64) at 1/2/4/8 B200; % of HBM roofline"

# (stencil, space, equilibrium, zero_centered, precision, streaming, shape(N), rates, description)
CONFIGS = {
    "c4": dict(stencil=W.D3Q27, space=W.CUMULANT, eq=W.EQ_ABSOLUTE, zc=1, prec=0, streaming=0,
               shape=lambda n: (1024, 1024, 128 * n), slab=2,
               desc="D3Q27 cumulant TGV 1024x1024x(128*N) z-slabs, fp64, zero-centered + absolute eq, pull"),
    "c4aa": dict(stencil=W.D3Q27, space=W.CUMULANT, eq=W.EQ_ABSOLUTE, zc=1, prec=0, streaming=1,
                 shape=lambda n: (1024, 1024, 128 * n), slab=2,
                 desc="D3Q27 cumulant TGV 1024x1024x(128*N) z-slabs, fp64, zero-centered + absolute eq, "
                      "AA in-place (one grid)"),
    "c4_strong": dict(stencil=W.D3Q27, space=W.CUMULANT, eq=W.EQ_ABSOLUTE, zc=1, prec=0, streaming=1,
                      shape=lambda n: (1024, 1024, 1024), slab=2, scaling="strong",
                      desc="D3Q27 cumulant TGV 1024^3 (strong scaling, N >= 2: 232 GB in AA), fp64, "
                           "zero-centered + absolute eq, AA in-place"),
    "c3": dict(stencil=W.D3Q27, space=W.CENTRAL, eq=W.EQ_ABSOLUTE, zc=1, prec=0, streaming=1,
               shape=lambda n: (384, 384, 384), slab=2, scaling="strong",
               desc="D3Q27 central-moment MRT TGV 384^3, fp64, zero-centered + absolute eq, AA in-place"),
    "c3eso": dict(stencil=W.D3Q27, space=W.CENTRAL, eq=W.EQ_ABSOLUTE, zc=1, prec=0, streaming=2,
                  shape=lambda n: (384, 384, 384), slab=2, scaling="strong",
                  desc="D3Q27 central-moment MRT TGV 384^3, fp64, zero-centered + absolute eq, Esoteric Pull"),
    "c3twist": dict(stencil=W.D3Q27, space=W.CENTRAL, eq=W.EQ_ABSOLUTE, zc=1, prec=0, streaming=3,
                    shape=lambda n: (384, 384, 384), slab=2, scaling="strong",
                    desc="D3Q27 central-moment MRT TGV 384^3, fp64, zero-centered + absolute eq, Esoteric Twist"),
    "c3push": dict(stencil=W.D3Q27, space=W.CENTRAL, eq=W.EQ_ABSOLUTE, zc=1, prec=0, streaming=4,
                   shape=lambda n: (384, 384, 384), slab=2, scaling="strong",
                   desc="D3Q27 central-moment MRT TGV 384^3, fp64, zero-centered + absolute eq, Esoteric Push"),
    "c4disc": dict(stencil=W.D3Q27, space=W.CUMULANT, eq=W.EQ_DISCRETE, zc=1, prec=0, streaming=0,
                   shape=lambda n: (1024, 1024, 128 * n), slab=2, scaling="weak",
                   desc="D3Q27 cumulant TGV 1024x1024x(128*N), fp64, zero-centered, DISCRETE f_eq (R29), pull"),
    "c3disc": dict(stencil=W.D3Q27, space=W.CENTRAL, eq=W.EQ_DISCRETE, zc=1, prec=0, streaming=1,
                   shape=lambda n: (384, 384, 384), slab=2, scaling="strong",
                   desc="D3Q27 central-moment MRT TGV 384^3, fp64, zero-centered, DISCRETE f_eq (R29), AA"),
    "c2_f64": dict(stencil=W.D3Q19, space=W.RAW, eq=W.EQ_DELTA, zc=1, prec=0, streaming=0,
                   shape=lambda n: (256, 256, 256), slab=2, scaling="strong",
                   desc="D3Q19 raw-moment MRT TGV 256^3, fp64, zero-centered + delta eq, pull"),
    "c2_f32": dict(stencil=W.D3Q19, space=W.RAW, eq=W.EQ_DELTA, zc=1, prec=1, streaming=0,
                   shape=lambda n: (256, 256, 256), slab=2, scaling="strong",
                   desc="D3Q19 raw-moment MRT TGV 256^3, fp32, zero-centered + delta eq, pull"),
    "c1": dict(stencil=W.D2Q9, space=W.POPULATION, eq=W.EQ_DELTA, zc=1, prec=0, streaming=0,
               shape=lambda n: (64, 64, 1), slab=1, scaling="strong", steps=1000,
               desc="D2Q9 BGK TGV 64x64, fp64, zero-centered + delta eq, pull"),
    "c5": dict(stencil=W.D2Q9, space=W.CENTRAL, eq=W.EQ_SWE, zc=0, prec=0, streaming=0,
               shape=lambda n: (8192, 8192, 1), slab=1, scaling="strong",
               desc="D2Q9 shallow-water CM LBM (Zhou eq.) dam break 8192^2, fp64, absolute, pull"),
    "c5zc": dict(stencil=W.D2Q9, space=W.CENTRAL, eq=W.EQ_SWE, zc=1, prec=0, streaming=0,
                 shape=lambda n: (8192, 8192, 1), slab=1, scaling="strong",
                 desc="D2Q9 shallow-water CM LBM (Zhou eq.) dam break 8192^2, fp64, zero-centered about the "
                      "rest state (R33), pull"),
}


def bytes_per_cell(cfg):
    q = W.Q_OF[cfg["stencil"]]
    return 2 * q * (8 if cfg["prec"] == 0 else 4)


def rates_of(cfg):
    st = cfg["stencil"]
    if cfg["space"] == W.POPULATION:
        return np.array([1.6])
    if cfg["eq"] == W.EQ_SWE:
        return W.regularized_rates(st, W.swe_lattice_parameters()[2])
    return W.rate_set_p(st)


def dtype_name(cfg):
    return "f64" if cfg["prec"] == 0 else "f32"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_name, kernel_key, cells, steps_per_launch=1):
    """Per-launch DRAM bytes (read + write) of the timed kernel from the committed
    ncu --set full capture (profiles/ncu_summary.json: bytes per cell of the same
    kernel, single-step or two fused steps) times this launch's cells, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as fh:
            d = json.load(fh)
        e = d.get(config_name)
        if e and e.get("kernel_key") == kernel_key and int(e.get("time_steps_per_launch", 1)) == steps_per_launch:
            return round(float(e["dram_bytes_per_cell"]) * cells)
    except Exception:
        return None
    return None


def global_sums(lat, n, dist):
    """mass and momentum of the whole lattice (lbm_get_diagnostics of every rank's slab,
    all-reduced in fp64)."""
    d = lat.get_diagnostics()
    v = np.array([d["mass"], *d["momentum"]], dtype=np.float64)
    if n > 1:
        import torch

        t = torch.from_numpy(v).to("cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t)
        v = t.cpu().numpy()
    return v


def multi_rank_probe(cfg, n, rank, dev, dist, L, D, use_nccl, want_peer):
    """N ranks vs rank 0 alone on a small lattice of the same method and halo path: every rank
    runs its slab of (64, 64, 8 N) (2D: (256, 16 N)) for 6 steps; rank 0 also runs the whole
    lattice as one rank and compares the gathered populations.  Returns (bitwise, max |diff|)
    on rank 0 (None elsewhere).  The first multi-GPU run proves its own halos."""
    st = cfg["stencil"]
    two_d = W.DIM_OF[st] == 2
    shape = (256, 16 * n, 1) if two_d else (64, 64, 8 * n)
    rates = rates_of(cfg)
    g = W.swe_lattice_parameters()[0] if cfg["eq"] == W.EQ_SWE else 0.0
    kw = dict(zero_centered=cfg["zc"], precision=cfg["prec"], streaming=cfg["streaming"], swe_g=g, device=dev)
    nid = None
    if use_nccl:
        box = [L.nccl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        nid = box[0]
    lat = L.Lattice(st, cfg["space"], cfg["eq"], rates, shape, rank=rank, nranks=n, nccl_id=nid, **kw)
    nx, ny, nz = shape
    if cfg["eq"] == W.EQ_SWE:
        rho, u = W.dam_break_fields(nx, ny, nx * 2.5 / 40, 6.25, 1.25, y0=lat.offset, ny_local=lat.extent)
    elif two_d:
        rho_g, u_g = W.tgv_fields(nx, ny, 1, 0.05)
        rho, u = rho_g[:, lat.offset:lat.offset + lat.extent], u_g[:, :, lat.offset:lat.offset + lat.extent]
    else:
        rho, u = W.tgv_fields(nx, ny, lat.extent, 0.05, z0=lat.offset, nz_global=nz, plane="xz")
    lat.init_macroscopic(np.ascontiguousarray(rho), np.ascontiguousarray(u[:lat.d]))
    runner = None
    if want_peer:
        try:
            runner = D.PeerRunner(lat, rank, n)
        except (L.LbmError, D.PeerUnavailable):
            runner = None
    if runner is None and not use_nccl:
        runner = D.SlabRunner(lat, rank, n)
        runner.prime()
    steps = 6
    (runner.step if runner is not None else lat.step)(steps)
    lat.sync()
    mine = lat.get_populations()
    parts = [None] * n
    dist.all_gather_object(parts, mine)
    dist.barrier()
    lat.close()
    if rank != 0:
        return None, None
    got = np.concatenate(parts, axis=2 if two_d else 1)
    with L.Lattice(st, cfg["space"], cfg["eq"], rates, shape, **kw) as one:
        rho, u = (W.dam_break_fields(nx, ny, nx * 2.5 / 40, 6.25, 1.25) if cfg["eq"] == W.EQ_SWE else
                  (W.tgv_fields(nx, ny, 1, 0.05) if two_d else W.tgv_fields(nx, ny, nz, 0.05, plane="xz")))
        one.init_macroscopic(np.ascontiguousarray(rho), np.ascontiguousarray(u[:one.d]))
        one.step(steps)
        ref = one.get_populations()
    return bool(np.array_equal(got, ref)), float(np.max(np.abs(got - ref)))


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi has printed its first sample (NVML start-up can take longer
        than a short timed region), so the region is always bracketed by samples."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)

    def stop(self):
        if not self.proc:
            return None
        if not self.lines:
            self.wait_first(2.0)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for k, name in enumerate(names):
                if parts[5 + k].lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
def oracle_mlups(cfg, target_seconds=15.0, max_cells=None):
    """Time the CPU oracle (fp64 instantiation, as it stands) on a bounded sample of
    the same workload: a periodic TGV box with the config's method.  Returns
    (mlups, cores, sample description)."""
    import oracle

    # every host core (torchrun exports OMP_NUM_THREADS=1 to its ranks)
    oracle.set_threads(len(os.sched_getaffinity(0)))
    st = cfg["stencil"]
    q = W.Q_OF[st]
    rates = rates_of(cfg)
    g = W.swe_lattice_parameters()[0] if cfg["eq"] == W.EQ_SWE else 0.0
    two_d = W.DIM_OF[st] == 2

    def run(shape, steps):
        nx, ny, nz = shape
        if cfg["eq"] == W.EQ_SWE:
            rho, u = W.dam_break_fields(nx, ny, nx * 2.5 / 40, 6.25, 1.25)
        else:
            rho, u = W.tgv_fields(nx, ny, nz, 0.05)
        feq = oracle.equilibrium(st, cfg["space"], cfg["eq"], cfg["zc"], rho.reshape(-1), u.reshape(3, -1).T, g=g)
        sim = oracle.Sim(st, cfg["space"], cfg["eq"], cfg["zc"], rates, shape, g=g, prec=oracle.DOUBLE)
        sim.set(np.ascontiguousarray(feq.T.reshape(q, nz, ny, nx)))
        t0 = time.perf_counter()
        sim.step(steps)
        return time.perf_counter() - t0

    probe = (64, 64, 1) if two_d else (64, 64, 4)
    t = run(probe, 1)
    cells = probe[0] * probe[1] * probe[2]
    per_cell = t / cells
    want = int(target_seconds / max(per_cell, 1e-12))
    if max_cells:
        want = min(want, max_cells)
    if two_d:
        ny = max(64, min(8192, (want // 1024) // 8 * 8))
        shape = (1024, ny, 1)
    else:
        nz = max(4, min(256, want // (256 * 256)))
        shape = (256, 256, nz)
    t = run(shape, 1)
    n = shape[0] * shape[1] * shape[2]
    return n / t / 1e6, oracle.max_threads(), f"1 step of a {shape[0]}x{shape[1]}x{shape[2]} periodic TGV box " \
                                                f"({n} cells), oracle fp64 instantiation (dense M/K(u), series cumulants)"


# ---------------------------------------------------------------------------
def reference_arm(args, cfg, name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle

    st = cfg["stencil"]
    q = W.Q_OF[st]
    rates = rates_of(cfg)
    g = W.swe_lattice_parameters()[0] if cfg["eq"] == W.EQ_SWE else 0.0
    # a bounded sample per step, sized by a probe so the whole --steps K --warmup W run ends in
    # a few minutes: <= 4 s per step and <= ~150 s for the K + W steps
    mlups0, cores, _ = oracle_mlups(cfg, target_seconds=2.0)
    per_step_s = min(4.0, max(0.05, 150.0 / max(1, args.steps + args.warmup)))
    per_step_cells = int(min(4e6, max(4096, mlups0 * 1e6 * per_step_s)))
    if W.DIM_OF[st] == 2:
        ny = max(64, (per_step_cells // 1024) // 8 * 8)
        shape = (1024, ny, 1)
    else:
        nz = max(4, per_step_cells // (256 * 256))
        shape = (256, 256, nz)
    nx, ny, nz = shape
    if cfg["eq"] == W.EQ_SWE:
        rho, u = W.dam_break_fields(nx, ny, nx * 2.5 / 40, 6.25, 1.25)
    else:
        rho, u = W.tgv_fields(nx, ny, nz, 0.05)
    feq = oracle.equilibrium(st, cfg["space"], cfg["eq"], cfg["zc"], rho.reshape(-1), u.reshape(3, -1).T, g=g)
    sim = oracle.Sim(st, cfg["space"], cfg["eq"], cfg["zc"], rates, shape, g=g, prec=oracle.DOUBLE)
    sim.set(np.ascontiguousarray(feq.T.reshape(q, nz, ny, nx)))
    sim.step(args.warmup)
    t0 = time.perf_counter()
    sim.step(args.steps)
    dt = time.perf_counter() - t0
    cells = nx * ny * nz
    value = cells * args.steps / dt / 1e6
    sample = f"each step: one time step of a {nx}x{ny}x{nz} periodic box of the same method " \
             f"({cells} cells), oracle fp64 instantiation"
    line = {
        "impl": "reference", "metric": BASELINE_METRIC if name == "c4" else f"MLUPS ({cfg['desc']})",
        "value": value, "unit": "MLUPS", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": dtype_name(cfg), "data": "synthetic",
        "config": {"workload": cfg["desc"] + " (CPU oracle sample)", "sample_shape": [nx, ny, nz]},
        "cpu_baseline": {"value": value, "unit": "MLUPS", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: the workload's own count, C1 1000, else 100)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--backend", default=None, choices=["nccl", "gloo"],
                    help="torch.distributed backend for N > 1 (default: nccl with one GPU per rank)")
    ap.add_argument("--halo", default="auto", choices=["auto", "peer", "nccl", "exchange"],
                    help="N > 1 halo path: peer = boundary kernels store into (pull) or access (AA) "
                         "the neighbours' planes over NVLink peer memory; nccl = the library's own "
                         "NCCL send/recv in lbm_step; exchange = torch.distributed P2P driven from "
                         "Python; auto = peer, else nccl")
    ap.add_argument("--no-probe", action="store_true", help="skip the N-rank vs 1-rank bitwise probe")
    ap.add_argument("--shape", type=int, nargs=3, default=None,
                    help="override the global lattice shape (profiling runs only)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.steps is None:
        args.steps = cfg.get("steps", 100)
    if args.impl == "reference":
        return reference_arm(args, cfg, args.config)
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3

    import torch
    import torch.distributed as dist

    from paper_2211_02435_b200 import distributed as D
    from paper_2211_02435_b200 import lbm as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("launch with torchrun for --gpus > 1")
    ngpu = torch.cuda.device_count()
    dev = local_rank % ngpu  # ranks share a GPU only in functional checks (then gloo)
    torch.cuda.set_device(dev)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = args.backend or ("nccl" if ngpu >= world else "gloo")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    local_rank = dev
    n = world
    st = cfg["stencil"]
    q = W.Q_OF[st]
    shape = tuple(args.shape) if args.shape else cfg["shape"](n)
    nx, ny, nz = shape
    two_d = W.DIM_OF[st] == 2
    rates = rates_of(cfg)
    g = W.swe_lattice_parameters()[0] if cfg["eq"] == W.EQ_SWE else 0.0
    # a dedicated (non-default) stream: the library enqueues on it and the CUDA
    # events of the timed region are recorded on the same stream
    main_stream = torch.cuda.Stream()
    torch.cuda.set_stream(main_stream)
    use_nccl = n > 1 and dist.get_backend() == "nccl" and args.halo in ("auto", "nccl", "peer")
    want_peer = n > 1 and (args.halo == "peer" or (args.halo == "auto" and cfg["streaming"] in (L.LBM_PULL, L.LBM_AA)))
    probe = None
    if n > 1 and not args.no_probe:  # N ranks vs one rank, bitwise, before anything is timed
        bitwise, maxdiff = multi_rank_probe(cfg, n, rank, dev, dist, L, D, use_nccl, want_peer)
        # agreement to rounding is the bar (two-step pairs across ranks round differently from
        # the single rank's sweep); a fused peer push that misses it is not timed: the run falls
        # back to the library's NCCL exchange and probes that instead
        tol = 1e-12 if cfg["prec"] == 0 else 1e-5
        verdict = [bool(bitwise) or (maxdiff is not None and maxdiff <= tol)]
        dist.broadcast_object_list(verdict, src=0)
        fallback = None
        if not verdict[0] and want_peer and args.halo == "auto" and use_nccl:
            fallback = f"fused peer push failed the probe (max |diff| {maxdiff}); NCCL exchange timed"
            if rank == 0:
                print(f"warning: {fallback}", file=sys.stderr)
            want_peer = False
            bitwise, maxdiff = multi_rank_probe(cfg, n, rank, dev, dist, L, D, use_nccl, want_peer)
            verdict = [bool(bitwise) or (maxdiff is not None and maxdiff <= tol)]
            dist.broadcast_object_list(verdict, src=0)
        if not verdict[0]:
            raise RuntimeError(f"N-rank probe disagrees with the single rank: max |diff| {maxdiff}")
        probe = {"multi_rank_bitwise": bitwise, "multi_rank_max_abs_diff": maxdiff,
                 "multi_rank_tolerance": tol,
                 "probe": "6 steps of a (64, 64, 8 N) lattice (2D: 256 x 16 N), N ranks vs rank 0 alone"}
        if fallback:
            probe["probe_fallback"] = fallback
    nccl_id = None
    if use_nccl:  # in-library NCCL communicator (lbm_domain.nccl_id): the transport when no peer push
        box = [L.nccl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        nccl_id = box[0]
    lat = L.Lattice(st, cfg["space"], cfg["eq"], rates, shape, zero_centered=cfg["zc"], precision=cfg["prec"],
                    streaming=cfg["streaming"], swe_g=g, device=local_rank, stream=main_stream.cuda_stream,
                    rank=rank, nranks=n, nccl_id=nccl_id)
    d = lat.d
    # synthetic initial state of this rank's slab
    if cfg["eq"] == W.EQ_SWE:
        rho, u = W.dam_break_fields(nx, ny, nx * 2.5 / 40, 6.25, 1.25, y0=lat.offset, ny_local=lat.extent)
    elif two_d:
        rho_g, u_g = W.tgv_fields(nx, ny, 1, 0.05)
        rho = rho_g[:, lat.offset:lat.offset + lat.extent]
        u = u_g[:, :, lat.offset:lat.offset + lat.extent]
    else:
        rho, u = W.tgv_fields(nx, ny, lat.extent, 0.05, z0=lat.offset)
    rho = np.ascontiguousarray(rho)
    u = np.ascontiguousarray(u[:d])
    lat.init_macroscopic(rho, u)
    runner = None
    halo = None
    path = "single"
    if n > 1:
        if want_peer:
            try:
                D.PeerRunner(lat, rank, n)  # connects the ring; lbm_step then runs the fused push
                path = "peer"
                # device flags spun on by a one-thread kernel when every neighbour has its own GPU;
                # host-polled flags when ranks share a GPU (no kernel waits on another rank there)
                waits = "host-polled flags" if lat.info().peer_wait_host else "device flags"
                halo = (f"peer: fused boundary-plane push over NVLink peer memory (CUDA IPC), {waits}, "
                        "lbm_step" if cfg["streaming"] == L.LBM_PULL else
                        "peer: AA odd-step boundary kernels access the neighbours' planes over NVLink peer "
                        f"memory (CUDA IPC), {waits}, lbm_step")
            except (L.LbmError, D.PeerUnavailable) as ex:
                if args.halo == "peer":
                    raise
                print(f"warning: fused halo push unavailable ({ex}); using the NCCL exchange", file=sys.stderr)
        if path == "single" and nccl_id is not None:
            path = "nccl"
            halo = "nccl: in-library ncclSend/ncclRecv group per step (lbm_step), overlapped with the interior"
        elif path == "single":
            path = "exchange"
            runner = D.SlabRunner(lat, rank, n)
            runner.prime()
            halo = f"exchange: torch.distributed P2P ({dist.get_backend()}) overlapped with the interior"

    def do_steps(k):  # the library's own collective lbm_step on every path but the external one
        if runner is None:
            lat.step(k)
        else:
            runner.step(k)

    cells_local = lat.cells
    # warm-up
    do_steps(args.warmup)
    torch.cuda.synchronize()
    sums0 = global_sums(lat, n, dist)
    if n > 1:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    sampler.wait_first()
    time.sleep(0.15)
    # the K timed steps in (up to) 5 windows of consecutive steps, CUDA events between them
    nwin = max(1, min(5, args.steps))
    # window edges on multiples of the steps one launch fuses (lbm_step runs whole sweeps inside
    # a window; the remainder of K goes to the last window)
    fuse = max(1, lat.info().temporal_blocking) if n == 1 else 1
    bounds = [0] + [min(args.steps, round(k * args.steps / nwin / fuse) * fuse) for k in range(1, nwin)] + [args.steps]
    bounds = sorted(set(bounds))
    nwin = len(bounds) - 1
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(nwin + 1)]
    torch.cuda.synchronize()
    if n > 1:
        dist.barrier()
    evs[0].record(main_stream)
    for k in range(nwin):
        do_steps(bounds[k + 1] - bounds[k])
        evs[k + 1].record(main_stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = evs[0].elapsed_time(evs[-1])
    win_ms = [evs[k].elapsed_time(evs[k + 1]) / (bounds[k + 1] - bounds[k]) for k in range(nwin)]
    def max_over_ranks(v):
        if n == 1:
            return v
        on_gpu = dist.get_backend() == "nccl"
        t = torch.tensor([v], device="cuda" if on_gpu else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ms)
    win_ms = [max_over_ranks(w) for w in win_ms]
    if n > 1:
        if path == "peer" and lat.peer_timed_out():
            raise RuntimeError(f"rank {rank}: a wait for a neighbour's halo timed out")
        dist.barrier()
    lat.check_finite()
    # conservation over the timed steps (periodic box: mass and momentum are invariants)
    sums1 = global_sums(lat, n, dist)
    mass_drift = float(abs(sums1[0] - sums0[0]) / sums0[0])
    momentum_drift = float(np.max(np.abs(sums1[1:] - sums0[1:])) / sums0[0])
    drift_tol = 1e-12 if cfg["prec"] == 0 else 1e-9
    if not (mass_drift <= drift_tol and momentum_drift <= drift_tol):
        raise RuntimeError(f"conservation violated over the timed steps: mass {mass_drift:.3e}, "
                           f"momentum {momentum_drift:.3e} (tolerance {drift_tol:g})")
    total_cells = nx * ny * nz
    value = total_cells * args.steps / (ms * 1e-3) / 1e6
    ms_step = ms / args.steps

    # dominant kernel: the stream–collide kernel (one launch per step at N = 1, or one launch
    # per TWO steps when the library fuses pairs of steps: temporal blocking, D3Q19)
    peak, peak_src = measured_peaks()
    bpc = bytes_per_cell(cfg)  # every population read once and written once per launch
    info = lat.info()
    tb = info.temporal_blocking
    if path == "exchange" and not runner.pairs:
        tb = 1
    resident = info.resident_cluster if n == 1 else 0
    # our kernels per step.  N > 1: interior + 2 boundary launches (+ wait and signal kernels of
    # the fused push; NCCL's own kernels are not counted); per PAIR of steps with two-step sweeps
    # across ranks: interior sweep + 4 boundary (+ 2 waits + 2 signals on the peer path)
    if n == 1:
        launches_per_step = 1.0 / tb
    elif path == "peer":  # per sweep: interior + 2 boundary launches, a wait and a signal per phase
        launches_per_step = {1: 5.0, 2: 4.5, 3: 13.0 / 3.0}.get(tb, 5.0)
        if lat.info().peer_wait_host:  # no wait kernels
            launches_per_step -= 1
    else:
        launches_per_step = 2.5 if tb == 2 else 3
    if resident:  # one cluster launch runs all K steps of lbm_step(K)
        launches_per_step = 1.0 / args.steps
    kernel_ms = ms_step * tb  # one launch covers tb steps on this stream
    achieved = bpc * cells_local / (kernel_ms * 1e-3) / 1e9
    kkey = f"{args.config}:{dtype_name(cfg)}"
    traffic = None if resident else ncu_traffic(args.config, kkey, cells_local, tb)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_source": ("scaled ncu capture: profiles/ncu_summary.json bytes per cell x cells per launch"
                                   if traffic is not None else None),
                "algorithmic_bytes_per_cell": bpc, "cells_per_launch": cells_local,
                "time_steps_per_launch": tb, "peak_source": peak_src,
                "kernel": ("k_pullD_2d (three fused steps)" if tb == 3 else
                           ("k_pull2_2d" if two_d else "k_pull2") + " (two fused steps)" if tb == 2 else
                           "k_pull/k_aa stream-collide") + f" ({kkey})"}
    if tb >= 2:
        # the single-step kernel's roofline, per time step: what the fused sweep beats
        roofline["frac_of_single_step_roofline_per_time_step"] = round(tb * achieved / peak, 4)
        roofline["note"] = (f"{tb} fused steps per HBM sweep: the launch moves 2qS B/cell for {tb} updates; the "
                            "sweep is bound by the collision arithmetic at 2-3 CTAs/SM, not by HBM (ncu: fp64 "
                            "pipe 44 % C2 fp64, issue slots 70 % C2 fp32, fp64 pipe 61 % C5 two-step; "
                            "DESIGN.md 6.2b); K mod tb steps run as a pair / single step")
    if n > 1:
        roofline["note"] = "N > 1: per-step time of boundary + interior launches with the halo " + halo.split(":")[0]
    if resident:
        roofline["kernel"] = f"k_resident2 (cluster of {resident} CTAs, lattice in shared memory) ({kkey})"
        roofline["note"] = ("cluster-resident loop: HBM is touched once per launch, a step is bound by the "
                            "collision latency, a DSMEM store and one cluster barrier; achieved = the "
                            "algorithmic bytes a step would move / step time, for comparison only")

    # end-to-end through the C ABI with host buffers (pinned): init from host rho/u,
    # K steps, macroscopic fields back to the host
    e2e = None
    if not args.no_e2e:
        rho_h = torch.from_numpy(rho.reshape(-1)).pin_memory()
        u_h = torch.from_numpy(u.reshape(-1)).pin_memory()
        rho_o = torch.empty_like(rho_h).pin_memory()
        u_o = torch.empty_like(u_h).pin_memory()
        import ctypes

        dp = ctypes.POINTER(ctypes.c_double)
        Lb = L.lib()
        torch.cuda.synchronize()
        if n > 1:
            dist.barrier()
        t0 = time.perf_counter()
        st_ = Lb.lbm_init_macroscopic(lat._ctx, ctypes.cast(rho_h.data_ptr(), dp), ctypes.cast(u_h.data_ptr(), dp))
        assert st_ == 0
        if runner is not None:
            runner.prime()  # external exchange; lbm_step primes by itself after init
        do_steps(args.steps)
        st_ = Lb.lbm_get_macroscopic(lat._ctx, ctypes.cast(rho_o.data_ptr(), dp), ctypes.cast(u_o.data_ptr(), dp))
        assert st_ == 0
        torch.cuda.synchronize()
        dt = max_over_ranks(time.perf_counter() - t0)
        h2d = (rho_h.numel() + u_h.numel()) * 8 * n
        d2h = (rho_o.numel() + u_o.numel()) * 8 * n
        e2e = {"value": total_cells * args.steps / dt / 1e6, "unit": "MLUPS",
               "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
               "what": "lbm_init_macroscopic(host rho,u) + K x lbm_step + lbm_get_macroscopic(host rho,u), "
                       "pinned host buffers, wall clock"}

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu:
        try:
            v, cores, sample = oracle_mlups(cfg)
            cpu = {"value": v, "unit": "MLUPS", "cores": cores, "kind": "oracle", "sample": sample}
        except Exception as ex:  # report, never fail the bench on the baseline
            cpu = {"value": None, "unit": "MLUPS", "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}

    regs, local = lat.kernel_attributes()
    if rank == 0:
        line = {
            "metric": BASELINE_METRIC if args.config == "c4" else f"MLUPS ({cfg['desc']})",
            "value": round(value, 1), "unit": "MLUPS", "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": cfg.get("scaling", "weak"),
            "vs_baseline": None, "dtype": dtype_name(cfg), "data": "synthetic",
            "config": {"workload": cfg["desc"], "global_shape": [nx, ny, nz], "cells_per_gpu": cells_local,
                       "rates": "rate set P (SURVEY.md 8(d))" if cfg["space"] != W.POPULATION else "omega = 1.6",
                       "l2": "inputs larger than L2 (population grids >> 126 MB)" if cells_local * bpc > 1e9
                       else "small grid: L2-resident", "parallelism": f"z-slab x{n}" if n > 1 else "single GPU",
                       "kernel_regs": regs, "kernel_local_bytes": local,
                       **({"halo": halo} if halo else {})},
            "timing": {"windows": nwin, "ms_per_step_median": round(statistics.median(win_ms), 4),
                       "ms_per_step_min": round(min(win_ms), 4), "ms_per_step_max": round(max(win_ms), 4),
                       "spread": round((max(win_ms) - min(win_ms)) / statistics.median(win_ms), 4)},
            "conservation": {"mass_drift": mass_drift, "momentum_drift": momentum_drift, "tolerance": drift_tol,
                             "what": "|sum rho change| / sum rho and max |sum rho u change| / sum rho over "
                                     "the K timed steps, all ranks"},
            **(probe if probe else {}),
            "roofline": roofline,
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": int(math.ceil(launches_per_step * args.steps)),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if n > 1:
        dist.barrier()  # no rank frees grids a neighbour still maps (fused push)
    lat.close()
    if n > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
