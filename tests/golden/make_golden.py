"""Generates tests/golden/reference_mandelbrot.json by running the UNMODIFIED
reference (oracle/_ref/libcafx_ref.so, built from /root/reference/proj by
oracle/Makefile). Run here, in the container that has /root/reference; the
JSON is committed so the GPU box never needs the reference.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402

R = oracle.ref()
assert R is not None, "build the reference first: make -C oracle ref"

out = {"source": "oracle/_ref/libcafx_ref.so (reference proj/src compiled -O3 -DNDEBUG)",
       "run_mandelbrot": [], "cells": [], "rows": []}

# (16000, 500) is the paper's scale; ~30 s on 8 cores
for size, it in [(64, 50), (96, 60), (256, 100), (1024, 500), (2048, 500), (4096, 500),
                 (16000, 500)]:
    sums = set()
    for w in ([1, 2, 4, 8] if size <= 256 else [8]):
        sums.add(R.ref_run_mandelbrot(size, it, w, None))
    assert len(sums) == 1, (size, it, sums)
    out["run_mandelbrot"].append({"size": size, "max_iter": it, "checksum": str(sums.pop())})

for re, im, it in [(0.0, 0.0, 50), (0.0, 0.0, 500), (2.0, 0.0, 50), (0.0, 0.0, 100),
                   (2.0, 0.0, 100), (-2.0, 0.0, 50), (-0.75, 0.1, 1000), (-1.5, -1.0, 500),
                   (0.25, 0.0, 500), (-0.7436, 0.1318, 5000), (0.3, 0.5, 1000),
                   (-1.0, 0.3, 1), (1e-300, -1e-300, 64)]:
    out["cells"].append({"re": re, "im": im, "max_iter": it,
                         "count": int(R.ref_mandelbrot_cell(re, im, it))})

for y, size, it in [(128, 256, 100), (0, 64, 50), (63, 64, 50), (500, 1000, 200)]:
    row = np.empty(size, dtype=np.uint32)
    R.ref_mandelbrot_row(y, size, it, row.ctypes.data)
    out["rows"].append({"y": y, "size": size, "max_iter": it, "sum": int(row.sum()),
                        "fnv": str(oracle.fnv1a_u32(row)),
                        "counts": row.tolist() if size <= 256 else None})

path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_mandelbrot.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print("wrote", path)
