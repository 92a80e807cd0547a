"""Device-API 3xTF32 sgemm timing (CUDA events on the launching stream, split +
GEMM launches), n^3 for each n given; median and min of 10 after 3 warm-ups.
    python paper_1505_07368_b200/tools/sgemm_time.py 1024 16384
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402

with pkg.Context(1) as ctx:
    for n in [int(x) for x in sys.argv[1:]] or [1024]:
        A = torch.rand(n, n, device="cuda")
        B = torch.rand(n, n, device="cuda")
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
        print(json.dumps({"n": n, "pdl": os.environ.get("CAFXG_SGEMM_PDL", "1"),
                          "median_ms": round(statistics.median(ts), 4),
                          "min_ms": round(min(ts), 4),
                          "tflops_median": round(2 * n ** 3 / statistics.median(ts) / 1e9, 1)}))
        del A, B, C
