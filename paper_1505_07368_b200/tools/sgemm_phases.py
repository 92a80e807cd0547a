"""Where a 3xTF32 GEMM launch spends its time: per-CTA %globaltimer stamps at
fixed points of sgemm_3xtf32_kernel (the phase build, `make -C
paper_1505_07368_b200/csrc phases`), for one device-API GEMM after warm-up.

    CAFXG_LIB=build/phases/libcafxg_phases.so \
        python paper_1505_07368_b200/tools/sgemm_phases.py 1024 4096

Stamps (us after the split pass's first block started): 0 CTA start,
1 after griddepcontrol.wait (split done), 2 first stage landed (MMA warp),
3 last MMA issued, 4 chunk sums done (epilogue), 5 partial parked,
6 cluster barrier passed, 7 tile stored. Median / max over CTAs. Each CTA's
start is its %globaltimer; the later stamps are its own clock64 deltas
(converted with the CTA's start-to-end globaltimer span), since globaltimer
reads are too coarse to order events a microsecond apart.
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1505_07368_b200 as pkg  # noqa: E402
from paper_1505_07368_b200 import cafxg  # noqa: E402

NAMES = ["start", "dep_wait", "first_stage", "mma_issued", "chunks_summed", "parked",
         "cluster_sync", "stored"]

lib = cafxg.lib()
fn = lib.cafxg_debug_sgemm_phases
fn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
with pkg.Context(1) as ctx:
    for n in [int(x) for x in sys.argv[1:]] or [1024]:
        A = torch.rand(n, n, device="cuda")
        B = torch.rand(n, n, device="cuda")
        Cm = torch.empty(n, n, device="cuda")
        s = torch.cuda.Stream()
        runs = []
        for k in range(8):
            torch.cuda.synchronize()
            fn(None, 0, None, 1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ctx.sgemm_device(n, n, n, A.data_ptr(), B.data_ptr(), Cm.data_ptr(), s.cuda_stream,
                             mode=pkg.SGEMM_3XTF32)
            e1.record(s)
            torch.cuda.synchronize()
            ph = np.zeros((1024, 16), dtype=np.uint64)
            span = np.zeros(2, dtype=np.uint64)
            fn(ph.ctypes.data, 1024, span.ctypes.data, 0)
            if k < 3:
                continue
            used = ph[ph[:, 0] != 0].astype(np.int64)
            t0 = int(span[0]) if span[0] != np.uint64(2**64 - 1) else int(used[:, 0].min())
            gt, clk = used[:, :8], used[:, 8:]
            ns_per_clk = (gt[:, 7] - gt[:, 0]) / np.maximum(clk[:, 7] - clk[:, 0], 1)
            rel = np.where(clk != 0, (gt[:, :1] - t0) + (clk - clk[:, :1]) * ns_per_clk[:, None], 0)
            rel[:, 0] = gt[:, 0] - t0
            row = {"n": n, "ctas": int(len(used)), "event_us": round(e0.elapsed_time(e1) * 1e3, 2),
                   "split_us": round((int(span[1]) - t0) / 1e3, 2),
                   "clk_ghz": round(float(1 / np.median(ns_per_clk)), 3)}
            for i, name in enumerate(NAMES):
                col = rel[:, i][used[:, i] != 0]  # stamp taken in this run
                if len(col):
                    row[name] = [round(float(np.median(col)) / 1e3, 2), round(float(col.max()) / 1e3, 2)]
            runs.append(row)
        for r in runs:
            print(json.dumps(r), flush=True)
