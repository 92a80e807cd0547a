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

# host-side cost of the submit call itself (API calls, planning) vs the wait
import ctypes as C  # noqa: E402
with pkg.Context(1) as ctx:
    L = pkg.lib()
    for n in sizes:
        hA, hB = ctx.pinned_empty((n, n), np.float32), ctx.pinned_empty((n, n), np.float32)
        hC = ctx.pinned_empty((n, n), np.float32)
        d = pkg.SgemmDesc()
        d.M = d.N = d.K = n
        d.lda = d.ldb = d.ldc = n
        d.mode = pkg.SGEMM_AUTO
        from paper_1505_07368_b200.cafxg import DONE_FN  # noqa: E402
        noop = DONE_FN(lambda u, s: None)
        sub, tot = [], []
        for k in range(40):
            t0 = time.perf_counter()
            L.cafxg_sgemm_submit(ctx.handle, C.byref(d), hA.ctypes.data, hB.ctypes.data,
                                 hC.ctypes.data, noop, None)
            t1 = time.perf_counter()
            ctx.sync()
            t2 = time.perf_counter()
            if k >= 5:
                sub.append((t1 - t0) * 1e3)
                tot.append((t2 - t0) * 1e3)
        print(f"n={n} submit call {statistics.median(sub):.3f} ms, submit+sync "
              f"{statistics.median(tot):.3f} ms", flush=True)
        for h in (hA, hB, hC):
            ctx.pinned_free(h)
