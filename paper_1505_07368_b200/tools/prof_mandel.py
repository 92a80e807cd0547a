"""Small driver for ncu captures of the escape kernel: one warm-up and one
profiled launch of a BASELINE config through cafxg_mandelbrot_device.
    python paper_1505_07368_b200/tools/prof_mandel.py cfg3|cfg1|storm64|storm16|ref4096|ref16000
"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
if which == "cfg3":
    tiles = [pkg.mandel_desc(-0.75, -0.73, 0.10, 0.12, 16384, 16384, 1000)]
elif which == "cfg1":
    tiles = [pkg.mandel_desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100)]
elif which == "ref4096":
    tiles = [pkg.reference_desc(4096, 500)]
elif which == "ref16000":
    tiles = [pkg.reference_desc(16000, 500)]
else:  # storm64 / storm16: that many storm tiles in one launch
    tiles = []
    for k in range(int(which[5:] or 64)):
        x0, y0 = -2.0 + (k * 23 % 1472) / 512, -1.0 + (k * 37 % 960) / 512
        tiles.append(pkg.mandel_desc(x0, x0 + 0.125, y0, y0 + 0.125, 64, 64, 256, fp64=True,
                                     out_offset=k * 4096))
npx = sum(t.nrows * t.ncols for t in tiles)
out = torch.empty(npx, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
with pkg.Context(1) as ctx:
    for _ in range(2):
        ctx.mandelbrot_device(tiles, out.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
print(which, "iterations", int(out.to(torch.int64).sum()))
