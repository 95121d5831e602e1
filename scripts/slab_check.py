#!/usr/bin/env python
"""Multi-process z-slab check: N torch.distributed ranks (torchrun) step their slabs with
SlabRunner (boundary planes, halo exchange, interior planes on a second stream) and the
gathered result must equal a single-rank run of the whole lattice BITWISE.

Runs with NCCL when every rank has its own GPU, otherwise with gloo (ranks may share one
GPU; the halo blocks are then staged through pinned host memory).

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/slab_check.py
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import workloads as W  # noqa: E402
from paper_2211_02435_b200 import distributed as D  # noqa: E402
from paper_2211_02435_b200 import lbm as L  # noqa: E402

CASES = [
    ("D3Q27 K zc+eq", W.D3Q27, W.CUMULANT, W.EQ_ABSOLUTE, 1, (40, 12, 8)),
    ("D3Q19 RAW zc+delta walls", W.D3Q19, W.RAW, W.EQ_DELTA, 1, (36, 10, 8)),
    ("D2Q9 SWE CM", W.D2Q9, W.CENTRAL, W.EQ_SWE, 0, (48, 8, 1)),
    ("D3Q27 CM zc+eq AA", W.D3Q27, W.CENTRAL, W.EQ_ABSOLUTE, 1, (40, 12, 8)),
    ("D2Q9 K AA", W.D2Q9, W.CUMULANT, W.EQ_ABSOLUTE, 1, (48, 8, 1)),
    # two-step sweeps across ranks on the peer path (>= 6 planes per slab, tile-aligned x/y):
    # equal to the single-rank run to rounding, not bitwise
    ("D3Q19 RAW zc+delta TB", W.D3Q19, W.RAW, W.EQ_DELTA, 1, (32, 16, 8)),
]


def lattice_weights(st):
    """Lattice weights w_i [q, 1, 1, 1] (the zero-centered background), from the library's own
    velocity table: relative differences are taken on absolute populations."""
    xi, _ = L.stencil_info(st)
    n = np.abs(xi).sum(1)
    table = {W.D2Q9: [4 / 9, 1 / 9, 1 / 36], W.D3Q19: [1 / 3, 1 / 18, 1 / 36],
             W.D3Q27: [8 / 27, 2 / 27, 1 / 54, 1 / 216]}[st]
    return np.asarray([table[k] for k in n]).reshape(-1, 1, 1, 1)


def fields(st, eq, shape, z0, nzl):
    nx, ny, nz = shape
    if eq == W.EQ_SWE:
        h, u = W.dam_break_fields(nx, ny, 6.0, 6.25, 1.25, y0=z0, ny_local=nzl)
        return h, u[:2]
    if W.DIM_OF[st] == 2:
        r, u = W.tgv_fields(nx, ny, 1, 0.05)
        return r[:, z0:z0 + nzl], u[:2, :, z0:z0 + nzl]
    r, u = W.tgv_fields(nx, ny, nzl, 0.05, plane="xz", z0=z0, nz_global=nz)
    return r, u


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--halo", choices=["exchange", "peer"], default="exchange",
                    help="exchange: SlabRunner (NCCL/gloo P2P); peer: PeerRunner (fused push over CUDA IPC)")
    ap.add_argument("--suballoc", action="store_true",
                    help="population grids from a torch-backed dev_alloc that returns pointers 4 KiB inside "
                         "their blocks (the peer path must map them at their offset)")
    args = ap.parse_args()
    # the TB case's small slabs keep their two-step sweeps (below the 2-wave rule of lbm_create)
    os.environ.setdefault("LBM_PEER_TB", "1")
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ngpu = torch.cuda.device_count()
    dev = local % ngpu
    torch.cuda.set_device(dev)
    backend = "nccl" if ngpu >= world else "gloo"
    dist.init_process_group(backend)
    ok = True
    for name, st, space, eq, zc, base in CASES:
        nx, ny, nz = base
        shape = (nx, ny * world, 1) if W.DIM_OF[st] == 2 else (nx, ny, nz * world)
        g = W.swe_lattice_parameters()[0] if eq == W.EQ_SWE else 0.0
        rates = W.regularized_rates(st, 1.3) if eq == W.EQ_SWE else W.rate_set_p(st)
        bc = None
        if "walls" in name:
            bc = [[0, 0], [0, 0], [L.LBM_BC_NOSLIP, L.LBM_BC_NOSLIP]]
        streaming = L.LBM_AA if name.endswith("AA") else L.LBM_PULL
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        allocator = None
        if args.suballoc:
            blocks = {}

            def alloc(nbytes, blocks=blocks):
                t = torch.empty(nbytes + 8192, dtype=torch.uint8, device=f"cuda:{dev}")
                p = t.data_ptr() + 4096
                blocks[p] = t
                return p

            allocator = (alloc, lambda p, blocks=blocks: blocks.pop(p, None))
        lat = L.Lattice(st, space, eq, rates, shape, zero_centered=zc, bc=bc, swe_g=g, device=dev,
                        stream=stream.cuda_stream, rank=rank, nranks=world, streaming=streaming,
                        allocator=allocator)
        r, u = fields(st, eq, shape, lat.offset, lat.extent)
        lat.init_macroscopic(np.ascontiguousarray(r), np.ascontiguousarray(u[:lat.d]))
        runner = (D.PeerRunner if args.halo == "peer" else D.SlabRunner)(lat, rank, world)
        runner.prime()
        runner.step(args.steps)
        torch.cuda.synchronize()
        if args.halo == "peer":
            runner.check()
        mine = lat.get_populations()
        dist.barrier()  # no rank frees memory a neighbour still maps
        lat.close()
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        if rank == 0:
            axis = 2 if W.DIM_OF[st] == 2 else 1
            multi = np.concatenate(parts, axis=axis)
            with L.Lattice(st, space, eq, rates, shape, zero_centered=zc, bc=bc, swe_g=g, device=dev) as one:
                r, u = fields(st, eq, shape, 0, shape[1] if W.DIM_OF[st] == 2 else shape[2])
                one.init_macroscopic(np.ascontiguousarray(r), np.ascontiguousarray(u[:one.d]))
                one.step(args.steps)
                single = one.get_populations()
            if name.endswith("TB"):  # two-step sweeps across ranks (both transports): to rounding
                w = lattice_weights(st) if zc else 0.0
                same = bool(np.max(np.abs(multi - single) / np.abs(single + w)) < 1e-13)
            else:
                same = np.array_equal(multi, single)
            ok &= same
            print(f"[{backend} x{world} {args.halo}] {name} {shape}: {'PASS' if same else 'FAIL'} "
                  f"(max |diff| {np.abs(multi - single).max():.3e})", flush=True)
        dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("ALL PASS" if ok else "SOME FAILED", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
