"""Device-API 3xTF32 timing for arbitrary shapes (CUDA events, mean of 20):
    python paper_1505_07368_b200/tools/sgemm_shapes.py M,N,K [M,N,K ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402

shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(512, 1024, 1024)]
with pkg.Context(1) as ctx:
    s = torch.cuda.Stream()
    for M, N, K in shapes:
        A = torch.rand(M, K, device="cuda")
        B = torch.rand(K, N, device="cuda")
        C = torch.empty(M, N, device="cuda")
        torch.cuda.synchronize()
        for _ in range(3):
            ctx.sgemm_device(M, N, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                             mode=pkg.SGEMM_3XTF32)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            ctx.sgemm_device(M, N, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                             mode=pkg.SGEMM_3XTF32)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{M}x{N}x{K}: {ms * 1e3:.1f} us  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s", flush=True)
