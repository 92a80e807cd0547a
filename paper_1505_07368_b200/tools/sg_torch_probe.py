import sys, time, statistics, numpy as np
sys.path.insert(0, '.')
mode = sys.argv[1]
if mode != "plain":
    import torch
    torch.zeros(1, device="cuda")
import paper_1505_07368_b200 as pkg
from oracle import oracle
with pkg.Context(1) as ctx:
    n = 1024
    if mode == "torchdev":
        A = torch.rand(n, n, device="cuda"); B = torch.rand(n, n, device="cuda"); C = torch.empty(n, n, device="cuda")
        s = torch.cuda.Stream()
        for _ in range(20): ctx.sgemm_device(n, n, n, A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
    hA, hB, hC = (ctx.pinned_empty((n, n), np.float32) for _ in range(3))
    hA[...] = oracle.fill_uniform(n * n, 1).reshape(n, n); hB[...] = oracle.fill_uniform(n * n, 2).reshape(n, n)
    ctx.sgemm(hA, hB, hC)
    ts = []
    for _ in range(30):
        t = time.perf_counter(); ctx.sgemm(hA, hB, hC); ts.append((time.perf_counter() - t) * 1e3)
    print(mode, "median %.3f" % statistics.median(ts))
