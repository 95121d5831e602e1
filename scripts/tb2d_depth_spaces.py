#!/usr/bin/env python
"""Depth-3 vs depth-2 2D temporal blocking through lbm_step for every D2Q9 collision space
(8192^2, fp64 and fp32, TGV; CUDA events on the context stream, 60 steps after 6 warm-up):
MLUPS per LBM_TB_DEPTH.  python scripts/tb2d_depth_spaces.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2211_02435_b200 import lbm as L  # noqa: E402

n = 8192
rho, u = W.tgv_fields(n, n, 1, 0.05)
cases = [(W.POPULATION, W.EQ_DELTA, L.LBM_FP64), (W.RAW, W.EQ_DELTA, L.LBM_FP64), (W.CENTRAL, W.EQ_ABSOLUTE, L.LBM_FP64),
         (W.CUMULANT, W.EQ_ABSOLUTE, L.LBM_FP64), (W.POPULATION, W.EQ_DELTA, L.LBM_FP32),
         (W.CUMULANT, W.EQ_ABSOLUTE, L.LBM_FP32)]
for space, eq, prec in cases:
    rates = [1.6] if space == W.POPULATION else W.rate_set_p(W.D2Q9)
    res = {}
    for depth in ("2", "3"):
        os.environ["LBM_TB_DEPTH"] = depth
        with L.Lattice(W.D2Q9, space, eq, rates, (n, n, 1), zero_centered=True, precision=prec) as lat:
            lat.init_macroscopic(rho, np.ascontiguousarray(u[:2]))
            s = torch.cuda.ExternalStream(lat.stream)
            lat.step(6)
            lat.sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            lat.step(60)
            e1.record(s)
            e1.synchronize()
            res[depth] = (n * n * 60 / (e0.elapsed_time(e1) * 1e-3) / 1e6, lat.info().temporal_blocking,
                          lat.kernel_attributes()[0])
    print(f"space {space} eq {eq} prec {'f64' if prec == L.LBM_FP64 else 'f32'}: "
          + "  ".join(f"depth {d}: {v[0]:8.0f} MLUPS (tb {v[1]}, regs {v[2]})" for d, v in res.items())
          + f"  ratio {res['3'][0] / res['2'][0]:.3f}", flush=True)
