import sys, time, statistics, numpy as np
sys.path.insert(0, '.')
import paper_1505_07368_b200 as pkg
from paper_1505_07368_b200.shard import band_tiles
with pkg.Context(1) as ctx:
    full = pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 16384, 16384, 1000)
    for world in (8, 4, 2):
        tiles = band_tiles(full, world, 0, 64, global_offsets=False)
        npx = sum(t.nrows * t.ncols for t in tiles)
        h = ctx.pinned_empty(npx, np.uint32)
        ctx.mandelbrot(tiles, h)
        ts = []
        for _ in range(5):
            t = time.perf_counter(); ctx.mandelbrot(tiles, h); ts.append((time.perf_counter() - t) * 1e3)
        print(f"rank share 1/{world}: e2e median {statistics.median(ts):.3f} ms", flush=True)
        ctx.pinned_free(h)
