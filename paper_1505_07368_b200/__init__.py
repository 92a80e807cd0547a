"""cafx-b200: a B200-native backend for CAF's GPGPU compute-actor path.

The product is the C-ABI library ``libcafxg.so`` (include/cafxg.h) with
hand-written sm_100a kernels; this package holds its sources (``csrc/``) and
the ctypes binding (``cafxg``) used by the tests and bench.py.
"""
from .cafxg import (  # noqa: F401
    CENTRE, CORNER, FP32, FP64, SGEMM_3XTF32, SGEMM_AUTO, SGEMM_FFMA,
    CafxgError, ComputeActor, Context, MandelDesc, SgemmDesc, Tuning, kernel_signature, lib,
    mandel_desc, reference_desc, tile_pixels,
)

__all__ = [
    "CENTRE", "CORNER", "FP32", "FP64", "SGEMM_3XTF32", "SGEMM_AUTO", "SGEMM_FFMA",
    "CafxgError", "ComputeActor", "Context", "MandelDesc", "SgemmDesc", "Tuning",
    "kernel_signature", "lib", "mandel_desc", "reference_desc", "tile_pixels",
]
