"""Runs the cfg4 storm once with CAFXG_TRACE=1 to print the batch timeline."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import bench  # noqa: E402
import paper_1505_07368_b200 as pkg  # noqa: E402

with pkg.Context(1) as ctx:
    for closed in (False, False, True):
        r = bench.run_storm(ctx, closed_loop=closed)
        print({k: r[k] for k in ("mode", "wall_ms", "requests_per_s", "batches", "max_batch")},
              flush=True)
