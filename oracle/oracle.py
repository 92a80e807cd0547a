"""TEST INFRASTRUCTURE ONLY -- ctypes face of the CPU oracle.

Loaded by tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline
legs, never by the product package (``paper_1505_07368_b200``). The C sources
(``cafx_oracle.c``, ``sgemm_oracle.c``) cite the reference lines they restate;
``ref()`` opens the unmodified reference compiled by ``oracle/Makefile``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libcafx_ref.so")

FNV_SEED = 0xCBF29CE484222325


class OracleTile(C.Structure):
    _fields_ = [
        ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
        ("width", C.c_uint32), ("height", C.c_uint32),
        ("row0", C.c_uint32), ("nrows", C.c_uint32),
        ("col0", C.c_uint32), ("ncols", C.c_uint32),
        ("max_iter", C.c_uint32), ("precision", C.c_uint32), ("centre", C.c_uint32),
    ]


_lib = None
_ref = None


def build() -> None:
    """Compiles the oracle (and, when /root/reference exists, the reference)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.check_call(["make", "-s", "-C", HERE, "-j8", "ref"])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.check_call(["make", "-s", "-C", HERE, "all"])
        L = C.CDLL(LIB)
        u32, u64, f64, p = C.c_uint32, C.c_uint64, C.c_double, C.c_void_p
        L.oracle_cell_f64.restype = u32
        L.oracle_cell_f64.argtypes = [f64, f64, u32]
        L.oracle_cell_f32.restype = u32
        L.oracle_cell_f32.argtypes = [C.c_float, C.c_float, u32]
        L.oracle_coord.restype = f64
        L.oracle_coord.argtypes = [f64, f64, u32, u32, C.c_int]
        L.oracle_mandelbrot_row.argtypes = [u32, u32, u32, p]
        L.oracle_mandelbrot_tile.argtypes = [C.POINTER(OracleTile), p]
        L.oracle_mandelbrot_tile_mt.restype = u32
        L.oracle_mandelbrot_tile_mt.argtypes = [C.POINTER(OracleTile), p, u32, u32]
        L.oracle_fnv1a_u32.restype = u64
        L.oracle_fnv1a_u32.argtypes = [u64, p, C.c_size_t]
        L.oracle_run_mandelbrot.restype = u64
        L.oracle_run_mandelbrot.argtypes = [u32, u32, u32]
        L.oracle_fill_uniform.argtypes = [p, C.c_size_t, u64, u64, u32]
        L.oracle_uniform_at.restype = C.c_float
        L.oracle_uniform_at.argtypes = [u64, u64]
        L.oracle_sgemm_ref_rows.argtypes = [p, p, u32, u32, u32, u32, p, u32, p]
        L.oracle_sgemm_rel_err.restype = f64
        L.oracle_sgemm_rel_err.argtypes = [p, u32, p, u32, p, u32]
        L.oracle_sgemm_f32_mt.argtypes = [p, p, p, u32, u32, u32, u32, u32, u32, u32, u32, u32]
        _lib = L
    return _lib


def ref():
    """The unmodified reference (oracle/_ref/libcafx_ref.so), or None."""
    global _ref
    if _ref is None and os.path.exists(REF_LIB):
        R = C.CDLL(REF_LIB)
        R.ref_mandelbrot_cell.restype = C.c_uint32
        R.ref_mandelbrot_cell.argtypes = [C.c_double, C.c_double, C.c_uint32]
        R.ref_mandelbrot_row.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
        R.ref_run_mandelbrot.restype = C.c_uint64
        R.ref_run_mandelbrot.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.POINTER(C.c_double)]
        R.ref_region_iters_mt.restype = C.c_uint64
        R.ref_region_iters_mt.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double,
                                          C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.POINTER(C.c_double)]
        R.ref_tiles_mt.restype = C.c_uint64
        R.ref_tiles_mt.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint32,
                                   C.POINTER(C.c_double)]
        _ref = R
    return _ref


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---- Mandelbrot ---------------------------------------------------------------

def cell_f64(re: float, im: float, max_iter: int) -> int:
    return lib().oracle_cell_f64(re, im, max_iter)


def cell_f32(re: float, im: float, max_iter: int) -> int:
    return lib().oracle_cell_f32(re, im, max_iter)


def mandelbrot_row(y: int, size: int, max_iter: int) -> np.ndarray:
    out = np.empty(size, dtype=np.uint32)
    lib().oracle_mandelbrot_row(y, size, max_iter, _ptr(out))
    return out


def tile(x0, x1, y0, y1, width, height, max_iter, fp64, centre,
         row0=0, nrows=None, col0=0, ncols=None, threads=None,
         sample_stride=1) -> np.ndarray:
    """Counts of a generalised tile (rows x cols, row-major). With
    sample_stride > 1 only every sample_stride-th row is computed (others 0)."""
    nrows = height - row0 if nrows is None else nrows
    ncols = width - col0 if ncols is None else ncols
    t = OracleTile(x0, x1, y0, y1, width, height, row0, nrows, col0, ncols,
                   max_iter, 1 if fp64 else 0, 1 if centre else 0)
    out = np.zeros((nrows, ncols), dtype=np.uint32)
    threads = threads or os.cpu_count() or 1
    lib().oracle_mandelbrot_tile_mt(C.byref(t), _ptr(out), threads, sample_stride)
    return out


def ref_tiles(descs, n: int, threads=None):
    """The unmodified reference's mandelbrot_cell (fp64) over every pixel of
    `n` tile records laid out as cafxg_mandel_desc (a ctypes array or a buffer
    address): (packed counts, total iterations, seconds). None without
    oracle/_ref."""
    R = ref()
    if R is None:
        return None
    addr = descs if isinstance(descs, int) else C.addressof(descs)
    rec = (C.c_uint32 * (20 * n)).from_address(addr)
    dims = np.frombuffer(rec, dtype=np.uint32).reshape(n, 20)
    npx = int((dims[:, 11].astype(np.uint64) * dims[:, 13].astype(np.uint64)).sum())
    out = np.empty(npx, dtype=np.uint32)
    sec = C.c_double()
    it = R.ref_tiles_mt(addr, n, _ptr(out), threads or os.cpu_count() or 1, C.byref(sec))
    return out, int(it), sec.value


def fnv1a_u32(cells: np.ndarray, h: int = FNV_SEED) -> int:
    cells = np.ascontiguousarray(cells, dtype=np.uint32)
    return lib().oracle_fnv1a_u32(h, _ptr(cells), cells.size)


def run_mandelbrot(size: int, max_iter: int, threads: int | None = None) -> int:
    return lib().oracle_run_mandelbrot(size, max_iter, threads or os.cpu_count() or 1)


# ---- matmul -------------------------------------------------------------------

def fill_uniform(n: int, seed: int, offset: int = 0, threads=None) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    lib().oracle_fill_uniform(_ptr(out), n, seed, offset, threads or os.cpu_count() or 1)
    return out


def uniform_at(seed: int, idx: int) -> float:
    return lib().oracle_uniform_at(seed, idx)


def sgemm_ref_rows(A: np.ndarray, B: np.ndarray, rows, N: int, K: int,
                   lda: int | None = None, ldb: int | None = None) -> np.ndarray:
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    out = np.empty((rows.size, N), dtype=np.float64)
    lib().oracle_sgemm_ref_rows(_ptr(A), _ptr(B), N, K, lda or K, ldb or N,
                                _ptr(rows), rows.size, _ptr(out))
    return out


def sgemm_rel_err(C_: np.ndarray, R: np.ndarray, rows, N: int, ldc: int | None = None) -> float:
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    return lib().oracle_sgemm_rel_err(_ptr(C_), ldc or N, _ptr(R), N, _ptr(rows), rows.size)


def sgemm_f32(A, B, C_, N, K, row_begin, row_end, block=16, threads=None):
    lib().oracle_sgemm_f32_mt(_ptr(A), _ptr(B), _ptr(C_), N, K, K, N, N,
                              row_begin, row_end, block, threads or os.cpu_count() or 1)
