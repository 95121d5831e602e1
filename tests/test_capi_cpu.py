"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/lbm.h declares, and its host-only logic (argument validation,
admissibility, stencil convention, slab arithmetic) behaves as documented.
No compute call is made here (no GPU in CI)."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2211_02435_b200 as P
from paper_2211_02435_b200 import lbm as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "lbm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_]+\s*\*?\s*(lbm_[a-z_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = P.lib()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    # and the binding covers every declared function
    bound = {s[0] for s in L.SIGNATURES}
    assert set(names) == bound


def test_version():
    assert "sm_100a" in P.version()


@pytest.mark.parametrize("st", [L.LBM_D2Q9, L.LBM_D3Q19, L.LBM_D3Q27])
def test_stencil_convention_matches_oracle(st):
    """The library's velocity table follows the documented order, which the
    oracle derives independently from the written rule."""
    import oracle

    xi, opp = P.stencil_info(st)
    oxi, oopp, *_ = oracle.tables(st)
    np.testing.assert_array_equal(xi, oxi)
    np.testing.assert_array_equal(opp, oopp)


def test_slab_extent():
    assert P.slab_extent(128, 0, 4) == (0, 32)
    assert P.slab_extent(128, 3, 4) == (96, 32)
    with pytest.raises(P.LbmError):
        P.slab_extent(130, 0, 4)
    with pytest.raises(P.LbmError):
        P.slab_extent(128, 4, 4)


def create_status(**kw):
    """lbm_create status for a configuration (validation runs before any CUDA call)."""
    args = dict(stencil=L.LBM_D3Q27, space=L.LBM_SPACE_CUMULANT, eq=L.LBM_EQ_ABSOLUTE, zc=1,
                shape=(8, 8, 8), nrates=None, rates=None, precision=L.LBM_FP64, streaming=L.LBM_PULL,
                bc=None, rank=0, nranks=1)
    args.update(kw)
    q = L.Q_OF[args["stencil"]]
    n = args["nrates"] if args["nrates"] is not None else (1 if args["space"] == L.LBM_SPACE_POPULATION else q)
    rates = np.full(n, 1.2) if args["rates"] is None else np.asarray(args["rates"], np.float64)
    dom = L.lbm_domain()
    dom.nx, dom.ny, dom.nz = args["shape"]
    bc = args["bc"] or [[0, 0]] * 3
    for a in range(3):
        for s in range(2):
            dom.bc[a][s] = bc[a][s]
    dom.precision, dom.streaming = args["precision"], args["streaming"]
    dom.rank, dom.nranks = args["rank"], args["nranks"]
    h = ctypes.c_void_p()
    st = P.lib().lbm_create(args["stencil"], args["space"], args["eq"], rates.ctypes.data_as(L._dp), rates.size,
                            ctypes.byref(dom), args["zc"], ctypes.byref(h))
    if st == 0:
        P.lib().lbm_destroy(h)
    return st, P.lib().lbm_last_error(None).decode()


def test_admissibility_errors():
    """delta equilibria need zero-centered storage; cumulants
    are incompatible with delta equilibria."""
    st, msg = create_status(eq=L.LBM_EQ_DELTA, zc=0, space=L.LBM_SPACE_RAW)
    assert st == L.LBM_EUNSUPPORTED and "zero-centered" in msg
    st, msg = create_status(eq=L.LBM_EQ_DELTA, zc=1, space=L.LBM_SPACE_CUMULANT)
    assert st == L.LBM_EUNSUPPORTED and "cumulant" in msg
    st, _ = create_status(eq=L.LBM_EQ_SWE, stencil=L.LBM_D3Q27, space=L.LBM_SPACE_CENTRAL, zc=0)
    assert st == L.LBM_EUNSUPPORTED
    # zero-centered shallow water about the rest state (reading R33) passes validation
    st, _ = create_status(eq=L.LBM_EQ_SWE, stencil=L.LBM_D2Q9, space=L.LBM_SPACE_CENTRAL, zc=1, shape=(8, 8, 1))
    assert st != L.LBM_EUNSUPPORTED
    st, _ = create_status(eq=L.LBM_EQ_SWE, stencil=L.LBM_D2Q9, space=L.LBM_SPACE_RAW, zc=1, shape=(8, 8, 1))
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(streaming=L.LBM_ESOTERIC_PULL, nranks=2, rank=0)
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(streaming=L.LBM_ESOTERIC_PULL, bc=[[0, 0], [1, 1], [0, 0]])
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(streaming=L.LBM_ESOTERIC_TWIST, nranks=2, rank=0)
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(streaming=L.LBM_ESOTERIC_TWIST, bc=[[1, 1], [0, 0], [0, 0]])
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(streaming=L.LBM_ESOTERIC_PUSH, nranks=2, rank=0)
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(streaming=L.LBM_ESOTERIC_PUSH, bc=[[0, 0], [1, 1], [0, 0]])
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(streaming=5)
    assert st == L.LBM_EINVAL
    # discrete equilibrium (reading R29): its delta form needs zero-centered storage and is
    # incompatible with cumulants, like the continuous one
    st, _ = create_status(eq=L.LBM_EQ_DISCRETE_DELTA, zc=0, space=L.LBM_SPACE_RAW)
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(eq=L.LBM_EQ_DISCRETE_DELTA, zc=1, space=L.LBM_SPACE_CUMULANT)
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(eq=6)
    assert st == L.LBM_EINVAL
    # literal background-in-population-space form (reading R30): zero-centered only
    st, _ = create_status(eq=L.LBM_EQ_ABSOLUTE_F0, zc=0, space=L.LBM_SPACE_CENTRAL)
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(streaming=L.LBM_AA, bc=[[1, 1], [0, 0], [0, 0]], nranks=2, rank=0)
    assert st == L.LBM_EUNSUPPORTED
    st, _ = create_status(streaming=L.LBM_AA, bc=[[1, 1], [0, 0], [0, 0]])
    assert st != L.LBM_EUNSUPPORTED  # AA with walls on one rank passes validation


def test_argument_errors():
    assert create_status(nrates=5)[0] == L.LBM_EINVAL
    assert create_status(rates=np.full(27, 2.5))[0] == L.LBM_EINVAL
    assert create_status(rates=np.r_[np.full(26, 1.0), np.nan])[0] == L.LBM_EINVAL
    assert create_status(shape=(3, 8, 8))[0] == L.LBM_EINVAL
    assert create_status(stencil=L.LBM_D2Q9, space=L.LBM_SPACE_RAW, shape=(8, 8, 2))[0] == L.LBM_EINVAL
    assert create_status(nranks=3, rank=0)[0] == L.LBM_EINVAL  # 8 planes not divisible by 3
    assert create_status(nranks=8, rank=0)[0] == L.LBM_EINVAL  # 1-plane slabs
    assert create_status(bc=[[0, 1], [0, 0], [0, 0]])[0] == L.LBM_EINVAL  # half-periodic axis
    assert create_status(space=L.LBM_SPACE_POPULATION, nrates=27)[0] == L.LBM_EINVAL


def test_valid_create_needs_a_device(monkeypatch):
    """A valid configuration passes validation and then fails loudly without a GPU
    (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    st, msg = create_status()
    assert st == L.LBM_ECUDA, msg


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    monkeypatch.setattr(L, "_lib", None)
    monkeypatch.setattr(L, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        L.lib()


def test_binding_structs_match_the_header(tmp_path):
    """The ctypes structures of the binding have the C layout of include/lbm.h (size and
    every field offset), checked against a program gcc compiles from the header."""
    structs = {"lbm_domain": L.lbm_domain, "lbm_halo": L.lbm_halo, "lbm_layout": L.lbm_layout,
               "lbm_info": L.lbm_info, "lbm_diagnostics": L.lbm_diagnostics, "lbm_peer_info": L.lbm_peer_info}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "lbm.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for field in cls._fields_:
            f = field[0]
            lines.append(f'  printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    import subprocess

    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for field in cls._fields_:
            assert int(got[f"{name}.{field[0]}"]) == getattr(cls, field[0]).offset, (name, field[0])


def test_nccl_unique_id_without_gpu():
    """lbm_nccl_get_unique_id needs no GPU: it returns a 128-byte id, or LBM_ENCCL with a
    message when no libnccl.so.2 can be loaded (never a crash)."""
    import ctypes as C

    buf = C.create_string_buffer(128)
    st = L.lib().lbm_nccl_get_unique_id(buf)
    assert st in (L.LBM_OK, L.LBM_ENCCL)
    if st == L.LBM_OK:
        assert any(buf.raw)
    else:
        assert L.lib().lbm_last_error(None)
    assert L.lib().lbm_nccl_get_unique_id(None) == L.LBM_EINVAL
