"""Device-API 3xTF32 sgemm timing (CUDA events on the launching stream; one
fused launch per GEMM), n^3 for each n given; median and min of 10 after 3
warm-ups, plus a sampled-row error check.
    python paper_1505_07368_b200/tools/sgemm_time.py 1024 16384
"""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402
from oracle import oracle  # noqa: E402

with pkg.Context(1) as ctx:
    for n in [int(x) for x in sys.argv[1:]] or [1024]:
        A_h = oracle.fill_uniform(n * n, 1).reshape(n, n)
        B_h = oracle.fill_uniform(n * n, 2).reshape(n, n)
        A, B = torch.from_numpy(A_h).cuda(), torch.from_numpy(B_h).cuda()
        if os.environ.get("TRANSPOSE_B"):  # experiments: B handed over as B^T (K-major)
            B = B.t().contiguous()
        C = torch.empty(n, n, device="cuda")
        s = torch.cuda.Stream()
        ts = []
        for k in range(13):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(s)
            ctx.sgemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                             mode=pkg.SGEMM_3XTF32)
            b.record(s)
            torch.cuda.synchronize()
            if k >= 3:
                ts.append(a.elapsed_time(b))
        # back to back (as bench.py times cfg2): 20 launches between two
        # events, and the host's enqueue time per call
        reps = 20
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.sgemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                             mode=pkg.SGEMM_3XTF32)
        host_us = (time.perf_counter() - t0) / reps * 1e6
        b.record(s)
        torch.cuda.synchronize()
        b2b = a.elapsed_time(b) / reps
        rows = np.arange(0, n, max(1, n // 16), dtype=np.uint32)
        R = oracle.sgemm_ref_rows(A_h, B_h, rows, n, n)
        err = oracle.sgemm_rel_err(C.cpu().numpy(), R, rows, n)
        print(json.dumps({"n": n, "bn": os.environ.get("CAFXG_SGEMM_BN", "auto"),
                          "median_ms": round(statistics.median(ts), 4),
                          "min_ms": round(min(ts), 4), "b2b_ms": round(b2b, 4),
                          "host_us_per_call": round(host_us, 1),
                          "tflops_median": round(2 * n ** 3 / statistics.median(ts) / 1e9, 1),
                          "err": err}), flush=True)
        del A, B, C
