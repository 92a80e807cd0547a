"""Full-image parity of BASELINE cfg3 (16384^2 fp32, max_iter 1000, zoom):
every pixel from the GPU (host request through the C ABI) against the oracle
restatement computed with every host thread (test infrastructure). Slow on the
CPU side (~1-2 min on 16 cores); run on the GPU box and keep the log:
    python paper_1505_07368_b200/tools/full_parity_cfg3.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402
from oracle import oracle  # noqa: E402

W = H = 16384
REGION = (-0.75, -0.73, 0.10, 0.12)
with pkg.Context(1) as ctx:
    img = ctx.pinned_empty(W * H, np.uint32)
    t0 = time.perf_counter()
    ctx.mandelbrot(pkg.mandel_desc(*REGION, W, H, 1000), img)
    t1 = time.perf_counter()
    ref = oracle.tile(*REGION, W, H, 1000, fp64=False, centre=True)
    t2 = time.perf_counter()
    got = img.reshape(H, W)
    bad = int(np.count_nonzero(got != ref))
    print(f"cfg3 full image: {W * H} pixels, {bad} mismatches; GPU {1e3 * (t1 - t0):.1f} ms, "
          f"oracle {t2 - t0 - (t1 - t0):.1f} s on {os.cpu_count()} threads; "
          f"sum of counts {int(got.sum(dtype=np.uint64))} (GPU) "
          f"{int(ref.sum(dtype=np.uint64))} (oracle)", flush=True)
    ctx.pinned_free(img)
    sys.exit(1 if bad else 0)
