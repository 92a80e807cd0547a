import sys, time, statistics, numpy as np
sys.path.insert(0, '.')
import paper_1505_07368_b200 as pkg
with pkg.Context(1) as ctx:
    d = pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100)
    h = ctx.pinned_empty(1920 * 1080, np.uint32)
    for _ in range(5): ctx.mandelbrot(d, h)
    ts = []
    for _ in range(50):
        t = time.perf_counter(); ctx.mandelbrot(d, h); ts.append((time.perf_counter() - t) * 1e3)
    print("cfg1 e2e median %.4f min %.4f ms" % (statistics.median(ts), min(ts)))
