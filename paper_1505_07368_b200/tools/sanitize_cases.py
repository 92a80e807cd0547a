"""Small cases of every kernel for compute-sanitizer memcheck runs."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402

with pkg.Context(1) as ctx:
    # big-tile fp32/fp64 (coordinate tables), edges, multi-tile batch
    for w, h, it, fp64 in [(300, 200, 150, False), (97, 33, 600, True), (1, 1, 0, False),
                           (513, 3, 30, True)]:
        ctx.mandelbrot(pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, w, h, it, fp64=fp64))
    tiles = [pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 300, 200, 50 + 10 * k, fp64=bool(k & 1),
                             row0=k, nrows=7, col0=3 * k, ncols=40, out_offset=300 * k)
             for k in range(40)]
    ctx.mandelbrot(tiles, np.zeros(300 * 40, np.uint32))
    # actor batch of small tiles (inline coordinates, reply scatter)
    a = ctx.spawn("mandelbrot")
    outs = [ctx.pinned_empty(4096, np.uint32) for _ in range(64)]
    futs = [a.request([(pkg.MandelDesc * 1)(pkg.mandel_desc(-2 + k / 64, -2 + k / 64 + 0.125,
                                                             -1.0, -0.875, 64, 64, 256,
                                                             fp64=True))], outs[k])
            for k in range(64)]
    [f.result(60) for f in futs]
    # direct replies (one small request per batch): checked kernel, deferred
    # kernel with replays (fp32 and fp64), a multi-tile request
    for tiles in [[pkg.mandel_desc(-2.0, -1.875, -0.0625, 0.0625, 64, 64, 256, fp64=True)],
                  [pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 96, 80, 1000)],
                  [pkg.mandel_desc(-0.30, -0.20, 0.60, 0.70, 64, 48, 300, fp64=True)],
                  [pkg.mandel_desc(-1.0 + k / 8, -0.875 + k / 8, 0.0, 0.125, 64, 64, 256,
                                   fp64=True) for k in range(3)]]:
        out = ctx.pinned_empty(sum(t.nrows * t.ncols for t in tiles), np.uint32)
        a.request([(pkg.MandelDesc * len(tiles))(*tiles)], out).result(60)
        ctx.pinned_free(out)
    assert ctx.stats().direct_batches >= 4
    a.release()
    # sgemm: FFMA, 3xTF32 direct, pipelined host request; device FNV; run_mandelbrot
    for M, N, K, mode in [(100, 77, 33, pkg.SGEMM_FFMA), (256, 256, 64, pkg.SGEMM_3XTF32),
                          (1024, 256, 64, pkg.SGEMM_AUTO)]:
        A = np.random.default_rng(0).uniform(-1, 1, (M, K)).astype(np.float32)
        B = np.random.default_rng(1).uniform(-1, 1, (K, N)).astype(np.float32)
        ctx.sgemm(A, B, mode=mode)
    print(ctx.run_mandelbrot(96, 60))
print("sanitize cases ok")
