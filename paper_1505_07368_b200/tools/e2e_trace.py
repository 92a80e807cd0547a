import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1505_07368_b200 as pkg
with pkg.Context(1) as ctx:
    d = pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 16384, 16384, 1000)
    host = ctx.pinned_empty(16384*16384, np.uint32)
    ctx.mandelbrot(d, host)
    for _ in range(3):
        t = time.perf_counter(); ctx.mandelbrot(d, host); print("e2e ms", (time.perf_counter()-t)*1e3, flush=True)
