import os, sys
sys.path.insert(0, '.')
import bench
import paper_1505_07368_b200 as pkg
with pkg.Context(1) as ctx:
    bench.run_storm(ctx, closed_loop=True)
    st0 = ctx.stats()
    r = bench.run_storm(ctx, closed_loop=True)
    print({k: r[k] for k in ("wall_ms", "batches")}, flush=True)
