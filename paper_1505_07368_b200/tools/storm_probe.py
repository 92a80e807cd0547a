"""Open- and closed-loop request storms (BASELINE cfg4) back to back, three of
each after a warm-up, for A/B runs of runtime knobs:
    CAFXG_STATS=1 python paper_1505_07368_b200/tools/storm_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import bench  # noqa: E402
import paper_1505_07368_b200 as pkg  # noqa: E402

with pkg.Context(1) as ctx:
    for closed in [False, True, "scheduled"][int(os.environ.get("FIRST", "0")):]:
        bench.run_storm(ctx, closed_loop=closed)
        for _ in range(3):
            r = bench.run_storm(ctx, closed_loop=closed)
            print({k: r[k] for k in ("mode", "wall_ms", "batches", "mismatched_tiles")},
                  flush=True)
