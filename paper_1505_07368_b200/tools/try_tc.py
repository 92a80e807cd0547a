"""Quick check of the 3xTF32 tcgen05 path: error vs the fp64 oracle and
timing, through cafxg_sgemm_device. python .../try_tc.py [sizes...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402
from oracle import oracle  # noqa: E402

sizes = [int(x) for x in sys.argv[1:]] or [256, 1024, 4096]
with pkg.Context(1) as ctx:
    s = torch.cuda.Stream()
    for n in sizes:
        A = torch.from_numpy(oracle.fill_uniform(n * n, 1).reshape(n, n)).cuda()
        B = torch.from_numpy(oracle.fill_uniform(n * n, 2).reshape(n, n)).cuda()
        torch.cuda.synchronize()
        for mode, name in [(pkg.SGEMM_3XTF32, "3xtf32"), (pkg.SGEMM_FFMA, "ffma")]:
            C = torch.full((n, n), float("nan"), device="cuda")
            ctx.sgemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream,
                             mode=mode)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3 if n >= 8192 else 10
            e0.record(s)
            for _ in range(reps):
                ctx.sgemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                                 s.cuda_stream, mode=mode)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            rows = np.arange(0, n, max(1, n // 16), dtype=np.uint32)
            An, Bn, Cn = A.cpu().numpy(), B.cpu().numpy(), C.cpu().numpy()
            R = oracle.sgemm_ref_rows(An, Bn, rows, n, n)
            err = oracle.sgemm_rel_err(Cn, R, rows, n)
            print(f"n={n} {name}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s  err={err:.3e}  "
                  f"nan={int(np.isnan(Cn).sum())}", flush=True)
