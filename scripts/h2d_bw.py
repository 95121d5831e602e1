#!/usr/bin/env python
"""Pinned host<->device copy bandwidth of a 4.3 GB fp64 buffer (the C4 macroscopic fields) with 1-8
streams: the ceiling of bench.py's end-to-end number.  python scripts/h2d_bw.py"""
import torch, time
n = 4 * 134217728 * 8 // 8  # 4.3 GB of fp64
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
def run(k, direction):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize(); t = time.perf_counter()
    step = (n + k - 1) // k
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            a, b = i * step, min(n, (i + 1) * step)
            if direction == "h2d": d[a:b].copy_(h[a:b], non_blocking=True)
            else: h[a:b].copy_(d[a:b], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return n * 8 / dt / 1e9
for direction in ("h2d", "d2h"):
    for k in (1, 2, 4, 8):
        run(k, direction)
        print(direction, k, "streams", round(run(k, direction), 1), "GB/s", flush=True)
