"""Multi-process slab decomposition on the GPU box: torchrun launches 2 and 3 ranks
(sharing the box's GPU(s); gloo with host-staged halos when ranks share a device, NCCL
otherwise) through the product driver SlabRunner; the gathered state must equal the
single-rank run bitwise (scripts/slab_check.py)."""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nproc", [2, 3])
@pytest.mark.parametrize("halo", ["exchange", "peer"])
def test_torchrun_slabs_bitwise(nproc, halo):
    """halo=peer: the fused halo push across processes (CUDA IPC mappings of the
    neighbours' grids and flags; processes sharing one GPU order the phases on the host, no kernel spins)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "scripts", "slab_check.py"), "--steps", "9", "--halo", halo]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert "ALL PASS" in r.stdout


def test_torchrun_peer_push_suballocated_grids():
    """The fused halo push across processes when the population grids come from a dev_alloc
    that sub-allocates (pointers 4 KiB inside torch caching-allocator blocks): CUDA IPC maps
    whole blocks, so lbm_peer_info carries each grid's offset inside its block."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "scripts", "slab_check.py"), "--steps", "9", "--halo", "peer", "--suballoc"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert "ALL PASS" in r.stdout
