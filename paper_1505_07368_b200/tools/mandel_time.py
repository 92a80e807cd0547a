"""Device-resident timing of the escape kernel on a few workloads (CUDA events
on the launching stream, mean of 5 after 2 warm-ups). Run twice with
CAFXG_DEFERRED=0 / 1 to compare the per-step and the deferred escape test.
    python paper_1505_07368_b200/tools/mandel_time.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402


def storm(n, it, kx_min=0):
    rng = np.random.default_rng(7)
    tiles = []
    for k in range(n):
        kx, ky = int(rng.integers(kx_min, 1473)), int(rng.integers(0, 961))
        x0, y0 = -2.0 + kx / 512, -1.0 + ky / 512
        tiles.append(pkg.mandel_desc(x0, x0 + 0.125, y0, y0 + 0.125, 64, 64, it, fp64=True,
                                     out_offset=k * 4096))
    return tiles


WORK = {
    "cfg3_fp32_16384_it1000": [pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 16384, 16384, 1000)],
    "ref_fp64_16000_it500": [pkg.reference_desc(16000, 500)],
    "ref_fp64_4096_it500": [pkg.reference_desc(4096, 500)],
    "deep_fp32_4096_it5000": [pkg.mandel_desc(-0.7487, -0.7485, 0.0650, 0.0652, 4096, 4096,
                                              5000)],
    "storm_fp64_4096x64sq_it256": storm(4096, 256),
    "storm_fp64_16x64sq_it256": storm(16, 256),
    # the same storm with every tile at x >= -1.7 (all tiles clear of |c| ~ 2,
    # so the deferred escape test may serve the whole batch)
    "stormsafe_fp64_4096x64sq_it256": storm(4096, 256, kx_min=154),
    "storm_fp64_64x64sq_it256": storm(64, 256),
    "cfg1_fp32_1920x1080_it100": [pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100)],
    # cfg1's two host waves: the first 273 rows (512K pixels), then the rest
    "cfg1_wave0_rows0_273": [pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100, nrows=273)],
    "cfg1_wave1_rows273_1080": [pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100,
                                                row0=273)],
    # every pixel inside the main cardioid: no escapes, no replays (the main
    # loop alone)
    "inset_fp32_4096_it1000": [pkg.mandel_desc(-0.3, -0.1, -0.1, 0.1, 4096, 4096, 1000)],
    # cfg1's pitch without the columns near |c| = 2 (x >= -1.7: the deferred
    # escape test's safe box)
    "cfg1safe_fp32_1728x1080_it100": [pkg.mandel_desc(-1.7, 1.0, -1.0, 1.0, 1728, 1080, 100)],
    "tiny_fp32_64x64_it100": [pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 64, 64, 100)],
    "cfg1_middle_rows405_675": [pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100,
                                                row0=405, nrows=270)],
    "cfg3reg_fp32_4096_it3000": [pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 4096, 4096, 3000)],
    "deep_fp32_4096_it2000": [pkg.mandel_desc(-0.7487, -0.7485, 0.0650, 0.0652, 4096, 4096,
                                              2000)],
    "seahorse_fp64_4096_it2000": [pkg.mandel_desc(-0.76, -0.74, 0.09, 0.11, 4096, 4096, 2000,
                                                  fp64=True)],
}

only = sys.argv[1:] or list(WORK)
s = torch.cuda.Stream()
with pkg.Context(1) as ctx:
    for name in only:
        tiles = WORK[name]
        npx = sum(t.nrows * t.ncols for t in tiles)
        out = torch.empty(npx, dtype=torch.int32, device="cuda")
        ts = []
        for k in range(22):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(s)
            ctx.mandelbrot_device(tiles, out.data_ptr(), s.cuda_stream)
            b.record(s)
            torch.cuda.synchronize()
            if k >= 2:
                ts.append(a.elapsed_time(b))
        iters = int(out.cpu().numpy().view(np.uint32).sum(dtype=np.uint64))
        ms = sum(ts) / len(ts)
        print(json.dumps({"work": name, "deferred": os.environ.get("CAFXG_DEFERRED", "1"),
                          "ms": round(ms, 4), "giter_s": round(iters / ms / 1e6, 1),
                          "iters": iters}))
