"""cfg3 end to end through the C ABI (cafxg_mandelbrot into one pinned host
image), median of 5 after a warm-up; run under different CAFXG_WAVE_MPX /
CAFXG_MIN_WAVE_MPX to compare wave plans.
    python paper_1505_07368_b200/tools/cfg3_e2e_sweep.py
"""
import sys, time, statistics, numpy as np
sys.path.insert(0, '.')
import paper_1505_07368_b200 as pkg
with pkg.Context(1) as ctx:
    d = pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 16384, 16384, 1000)
    host = ctx.pinned_empty(16384*16384, np.uint32)
    ctx.mandelbrot(d, host)
    ts = []
    for _ in range(5):
        t = time.perf_counter(); ctx.mandelbrot(d, host); ts.append((time.perf_counter()-t)*1e3)
    print("e2e median %.3f min %.3f" % (statistics.median(ts), min(ts)), flush=True)
