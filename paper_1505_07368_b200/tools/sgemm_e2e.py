"""End-to-end host sgemm (cafxg_sgemm through the C ABI, pinned host A/B/C)
timing: median of N calls after warm-up, per size.
    python paper_1505_07368_b200/tools/sgemm_e2e.py [sizes...]"""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402
from oracle import oracle  # noqa: E402

sizes = [int(x) for x in sys.argv[1:]] or [1024, 2048]
with pkg.Context(1) as ctx:
    for n in sizes:
        hA, hB = ctx.pinned_empty((n, n), np.float32), ctx.pinned_empty((n, n), np.float32)
        hC = ctx.pinned_empty((n, n), np.float32)
        hA[:] = oracle.fill_uniform(n * n, 1).reshape(n, n)
        hB[:] = oracle.fill_uniform(n * n, 2).reshape(n, n)
        for _ in range(5):
            ctx.sgemm(hA, hB, hC)
        ts = []
        for _ in range(50 if n <= 2048 else 5):
            t0 = time.perf_counter()
            ctx.sgemm(hA, hB, hC)
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"n={n} e2e median {statistics.median(ts):.3f} ms  min {min(ts):.3f} ms", flush=True)
        for h in (hA, hB, hC):
            ctx.pinned_free(h)
