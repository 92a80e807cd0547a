"""One device-API 3xTF32 sgemm at n^3 (after warm-up) for profiling:
    python tc_once.py [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
with pkg.Context(1) as ctx:
    A = torch.rand(n, n, device="cuda")
    B = torch.rand(n, n, device="cuda")
    C = torch.empty(n, n, device="cuda")
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        ctx.sgemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                         mode=pkg.SGEMM_3XTF32)
    torch.cuda.synchronize()
