"""ncu driver for the direct-reply escape kernel: one 16-tile storm request
(64x64 fp64 tiles, max_iter 256) through the actor into a pinned reply, twice.
    ncu -k regex:mandel python paper_1505_07368_b200/tools/prof_direct.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402

rng = np.random.default_rng(7)
tiles = []
for k in range(16):
    kx, ky = int(rng.integers(0, 1473)), int(rng.integers(0, 961))
    x0, y0 = -2.0 + kx / 512, -1.0 + ky / 512
    tiles.append(pkg.mandel_desc(x0, x0 + 0.125, y0, y0 + 0.125, 64, 64, 256, fp64=True))
with pkg.Context(1) as ctx:
    a = ctx.spawn("mandelbrot")
    out = ctx.pinned_empty(16 * 4096, np.uint32)
    for _ in range(2):
        a.request([(pkg.MandelDesc * 16)(*tiles)], out).result(60)
    print("direct batches", ctx.stats().direct_batches, "iterations", int(out.sum()))
    ctx.pinned_free(out)
    a.release()
