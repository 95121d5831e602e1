#!/usr/bin/env python
"""Cost of the slab decomposition with the fused halo push, measured on ONE GPU: N slab
contexts of one process (cuda:0, lbm_peer_* over plain device pointers; since the
host-ordered waits, flags polled by the host as on any GPU shared by ranks — the round-1
numbers in profiles/r1/peer_overhead.txt were taken with device-side waits) step a 1024 x 1024 x 128 D3Q27 cumulant lattice together; compared with one context stepping
the whole lattice.  Same cells, same bytes: the difference is the boundary/interior split,
the wait/signal kernels and the halo stores.

  python scripts/peer_overhead.py [--steps 30] [--ranks 2 4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

# N contexts x 2 streams on ONE GPU: give every stream its own hardware queue, or a spinning
# neighbour-wait kernel can sit in front of another context's signal kernel in a shared queue
# (one process per GPU — the deployment case — uses two streams and never hits this)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2211_02435_b200 import distributed as D  # noqa: E402
from paper_2211_02435_b200 import lbm as L  # noqa: E402


CONFIG = "c4"


def make(shape, rank=0, nranks=1):
    if CONFIG == "c5":  # D2Q9 shallow water (CM, Zhou), dam break; slab axis = y
        st = W.D2Q9
        g, nu, om = W.swe_lattice_parameters()
        lat = L.Lattice(st, W.CENTRAL, W.EQ_SWE, W.regularized_rates(st, om), shape, zero_centered=False,
                        swe_g=g, rank=rank, nranks=nranks)
        h, u = W.dam_break_fields(shape[0], shape[1], shape[0] * 2.5 / 40, 6.25, 1.25, y0=lat.offset,
                                  ny_local=lat.extent)
        lat.init_macroscopic(np.ascontiguousarray(h), np.ascontiguousarray(u[:2]))
        return lat
    if CONFIG == "c2":  # D3Q19 raw moments, zc + delta
        st, space, eq = W.D3Q19, W.RAW, W.EQ_DELTA
    else:  # c4: D3Q27 cumulant
        st, space, eq = W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE
    lat = L.Lattice(st, space, eq, W.rate_set_p(st), shape, zero_centered=1, rank=rank, nranks=nranks)
    rho, u = W.tgv_fields(shape[0], shape[1], lat.extent, 0.05, z0=lat.offset)
    lat.init_macroscopic(np.ascontiguousarray(rho), np.ascontiguousarray(u))
    return lat


def timed(fn, steps, streams):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(streams[0])
    fn(steps)
    for s in streams[1:]:  # join every context stream into the first
        e = torch.cuda.Event()
        e.record(s)
        streams[0].wait_event(e)
    ev[1].record(streams[0])
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4])
    ap.add_argument("--shape", type=int, nargs=3, default=[1024, 1024, 128])
    ap.add_argument("--chunk", type=int, default=64,
                    help="steps per lbm_step_peer call (>= 32: captured CUDA graphs are replayed)")
    ap.add_argument("--config", default="c4", choices=["c4", "c2", "c5"])
    args = ap.parse_args()
    global CONFIG
    CONFIG = args.config
    shape = tuple(args.shape)
    cells = shape[0] * shape[1] * shape[2]
    out = {}
    lat = make(shape)
    s = [torch.cuda.ExternalStream(lat.stream)]
    lat.step(args.chunk)
    ms = timed(lambda k: [lat.step(min(args.chunk, k - i)) for i in range(0, k, args.chunk)], args.steps, s)
    out["1 context"] = ms
    out["1 context temporal_blocking"] = lat.info().temporal_blocking
    lat.close()
    for n in args.ranks:
        lats = [make(shape, r, n) for r in range(n)]
        D.connect_local(lats)
        streams = [torch.cuda.ExternalStream(l.stream) for l in lats]

        def run(k):
            # one host thread per context: on one GPU the peer phases are host-ordered
            # (lbm_info.peer_wait_host), no kernel waits on another context's flag
            def ctx(l):
                j = k
                while j > 0:
                    c = min(j, args.chunk)
                    l.step_peer(c)
                    j -= c
            D.on_ranks(lats, ctx)

        run(args.chunk)
        ms = timed(run, args.steps, streams)
        for l in lats:
            l.sync()
            assert not l.peer_timed_out()
        out[f"{n} slab contexts, fused push (temporal_blocking {lats[0].info().temporal_blocking})"] = ms
        for l in lats:
            l.close()
    base = out["1 context"]
    for k, v in out.items():
        if not isinstance(v, float):
            continue
        print(f"{k:32s} {v:7.3f} ms/step  {cells / v / 1e3:8.0f} MLUPS  overhead {100 * (v / base - 1):+5.1f} %")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
