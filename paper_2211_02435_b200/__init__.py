"""B200-native MRT lattice Boltzmann stream–collide (arXiv 2211.02435 hot path).

The product is liblbm.so (include/lbm.h): hand-written sm_100a CUDA kernels
behind a C ABI.  This package holds its thin Python binding (lbm.py), the
multi-rank slab driver (distributed.py) and the build script (build.py).
"""
from .lbm import *  # noqa: F401,F403
from .lbm import Lattice, LbmError, grid_layout, lib, slab_extent, stencil_info, version  # noqa: F401
