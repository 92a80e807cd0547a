"""Times the device FNV-1a and the fp64 reference-mode image separately."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402

n = 16000 * 16000
with pkg.Context(1) as ctx:
    s = torch.cuda.Stream()
    x = torch.randint(0, 1000, (n,), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    for _ in range(2):
        t = time.perf_counter()
        h = ctx.fnv1a_u32_device(x.data_ptr(), n, stream=s.cuda_stream)
        print(f"fnv {n} cells: {(time.perf_counter() - t) * 1e3:.2f} ms", flush=True)
    d = pkg.reference_desc(16000, 500)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ctx.mandelbrot_device(d, out.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"image fp64 16000^2 it=500: {e0.elapsed_time(e1):.2f} ms, "
              f"{out.to(torch.int64).sum().item() / e0.elapsed_time(e1) / 1e6:.1f} Giter/s",
              flush=True)
    for _ in range(2):
        print("run_mandelbrot", ctx.run_mandelbrot(16000, 500), flush=True)
