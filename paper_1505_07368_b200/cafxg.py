"""ctypes binding of libcafxg.so (include/cafxg.h).

This is the Python face the tests and bench.py call; every call goes through
the C ABI a CAF adapter (include/cafxg/gpu_actor.hpp) or any other FFI binds.
There is no CPU fallback: if the library or a B200 is missing, opening a
context raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from concurrent.futures import Future

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# CAFXG_LIB: another build of the library (A/B experiments, and the checked
# build with device-side bounds checks, tests/test_checked_build_gpu.py)
LIB_PATH = os.environ.get("CAFXG_LIB") or os.path.join(HERE, "libcafxg.so")

OK = 0
E_UNKNOWN_TYPE = 2
E_OUT_OF_RANGE = 4
E_TYPE_MISMATCH = 5
E_INTERFACE_MISMATCH = 6
E_CONFIG = 8
E_SPAWN = 9
E_TIMEOUT = 13
E_DOWN = 14

FP32, FP64 = 0, 1
CORNER, CENTRE = 0, 1
SGEMM_AUTO, SGEMM_FFMA, SGEMM_3XTF32 = 0, 1, 2

# Symbols include/cafxg.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "cafxg_abi_version", "cafxg_status_string", "cafxg_last_error",
    "cafxg_open", "cafxg_close", "cafxg_device_count", "cafxg_ctx_status", "cafxg_sync",
    "cafxg_host_alloc", "cafxg_host_free", "cafxg_host_register", "cafxg_host_unregister",
    "cafxg_mandelbrot_submit", "cafxg_mandelbrot", "cafxg_mandelbrot_device",
    "cafxg_fnv1a_u32_device", "cafxg_run_mandelbrot",
    "cafxg_sgemm_submit", "cafxg_sgemm", "cafxg_sgemm_device",
    "cafxg_spawn", "cafxg_spawn_ex", "cafxg_kernel_signature",
    "cafxg_actor_enqueue", "cafxg_actor_reply_bytes", "cafxg_completion_batch",
    "cafxg_actor_quit", "cafxg_actor_release", "cafxg_get_stats",
]


class CafxgError(RuntimeError):
    """A non-zero cafxg status; `code` is the cafx::errc value."""

    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {status_string(code)} ({code})")
        self.code = code


class MandelDesc(C.Structure):
    _fields_ = [
        ("x0", C.c_double), ("x1", C.c_double), ("y0", C.c_double), ("y1", C.c_double),
        ("width", C.c_uint32), ("height", C.c_uint32),
        ("row0", C.c_uint32), ("nrows", C.c_uint32),
        ("col0", C.c_uint32), ("ncols", C.c_uint32),
        ("max_iter", C.c_uint32), ("precision", C.c_uint32), ("sampling", C.c_uint32),
        ("reserved", C.c_uint32), ("out_offset", C.c_uint64),
    ]


class SgemmDesc(C.Structure):
    _fields_ = [("M", C.c_uint32), ("N", C.c_uint32), ("K", C.c_uint32),
                ("lda", C.c_uint32), ("ldb", C.c_uint32), ("ldc", C.c_uint32),
                ("mode", C.c_uint32), ("splits", C.c_uint32)]


class Tuning(C.Structure):
    """spawn_cl's tuning overload (cafxg_tuning): zero fields keep the
    backend's choice."""
    _fields_ = [("block_steps", C.c_uint32), ("max_ctas", C.c_uint32),
                ("sgemm_mode", C.c_uint32), ("sgemm_splits", C.c_uint32),
                ("reserved", C.c_uint32 * 4)]


class Stats(C.Structure):
    _fields_ = [("requests", C.c_uint64), ("batches", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("max_batch", C.c_uint64),
                ("direct_batches", C.c_uint64), ("nccl_collectives", C.c_uint64),
                ("devices_used", C.c_uint64), ("peer_gemms", C.c_uint64)]


DONE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int)

_lib = None


def lib() -> C.CDLL:
    """Loads libcafxg.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, sz, u64, i = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int
        L.cafxg_abi_version.restype = i
        L.cafxg_status_string.restype = C.c_char_p
        L.cafxg_status_string.argtypes = [i]
        L.cafxg_last_error.restype = C.c_char_p
        L.cafxg_open.argtypes = [u64, C.POINTER(vp)]
        L.cafxg_close.argtypes = [vp]
        L.cafxg_device_count.argtypes = [vp]
        L.cafxg_ctx_status.argtypes = [vp]
        L.cafxg_sync.argtypes = [vp]
        L.cafxg_host_alloc.argtypes = [vp, sz, C.POINTER(vp)]
        L.cafxg_host_free.argtypes = [vp, vp]
        L.cafxg_host_register.argtypes = [vp, vp, sz]
        L.cafxg_host_unregister.argtypes = [vp, vp]
        L.cafxg_mandelbrot_submit.argtypes = [vp, C.POINTER(MandelDesc), sz, vp, DONE_FN, vp]
        L.cafxg_mandelbrot.argtypes = [vp, C.POINTER(MandelDesc), sz, vp]
        L.cafxg_mandelbrot_device.argtypes = [vp, i, C.POINTER(MandelDesc), sz, vp, vp]
        L.cafxg_fnv1a_u32_device.argtypes = [vp, i, vp, u64, u64, C.POINTER(u64), vp]
        L.cafxg_run_mandelbrot.argtypes = [vp, C.c_uint32, C.c_uint32, C.POINTER(u64),
                                           C.POINTER(C.c_double)]
        L.cafxg_sgemm_submit.argtypes = [vp, C.POINTER(SgemmDesc), vp, vp, vp, DONE_FN, vp]
        L.cafxg_sgemm.argtypes = [vp, C.POINTER(SgemmDesc), vp, vp, vp]
        L.cafxg_sgemm_device.argtypes = [vp, i, C.POINTER(SgemmDesc), vp, vp, vp, vp]
        L.cafxg_spawn.argtypes = [vp, C.c_char_p, C.POINTER(u64), sz, C.POINTER(vp)]
        L.cafxg_spawn_ex.argtypes = [vp, C.c_char_p, C.c_char_p, C.POINTER(u64), sz,
                                     C.POINTER(Tuning), C.POINTER(vp)]
        L.cafxg_kernel_signature.argtypes = [C.c_char_p, C.c_char_p, sz]
        L.cafxg_actor_enqueue.argtypes = [vp, C.POINTER(vp), C.POINTER(sz), sz, vp, sz,
                                          DONE_FN, vp]
        L.cafxg_completion_batch.restype = sz
        L.cafxg_actor_reply_bytes.restype = sz
        L.cafxg_actor_reply_bytes.argtypes = [vp, C.POINTER(vp), C.POINTER(sz), sz]
        L.cafxg_actor_quit.argtypes = [vp]
        L.cafxg_actor_release.argtypes = [vp]
        L.cafxg_get_stats.argtypes = [vp, C.POINTER(Stats)]
        _lib = L
    return _lib


def status_string(code: int) -> str:
    return lib().cafxg_status_string(code).decode()


def last_error() -> str:
    return lib().cafxg_last_error().decode()


def _check(code: int, what: str) -> None:
    if code != OK:
        raise CafxgError(code, f"{what}: {last_error()}")


def mandel_desc(x0, x1, y0, y1, width, height, max_iter, fp64=False, centre=True,
                row0=0, nrows=None, col0=0, ncols=None, out_offset=0) -> MandelDesc:
    return MandelDesc(x0, x1, y0, y1, width, height, row0,
                      height - row0 if nrows is None else nrows, col0,
                      width - col0 if ncols is None else ncols, max_iter,
                      FP64 if fp64 else FP32, CENTRE if centre else CORNER, 0, out_offset)


def kernel_signature(kernel: str) -> str:
    """The kernel's normalised spawn_cl signature, e.g. "f32*(f32*,f32*)"."""
    buf = C.create_string_buffer(128)
    _check(lib().cafxg_kernel_signature(kernel.encode(), buf, 128), "kernel_signature")
    return buf.value.decode()


def reference_desc(size: int, max_iter: int) -> MandelDesc:
    """run_mandelbrot(size, max_iter)'s image (bench.cpp:381-390): fp64, corner
    sampling over [-1.5, 0.5] x [-1, 1]."""
    return mandel_desc(-1.5, 0.5, -1.0, 1.0, size, size, max_iter, fp64=True, centre=False)


def _desc_array(tiles):
    if isinstance(tiles, MandelDesc):
        tiles = [tiles]
    arr = (MandelDesc * len(tiles))(*tiles)
    return arr, len(tiles)


def tile_pixels(tiles) -> int:
    if isinstance(tiles, MandelDesc):
        tiles = [tiles]
    return sum(t.nrows * t.ncols for t in tiles)


class ComputeActor:
    """Handle of a `cafxg_spawn`ed compute actor (the spawn_cl facade)."""

    def __init__(self, ctx: "Context", handle: int, kernel: str):
        self.ctx, self.handle, self.kernel = ctx, handle, kernel
        self._keep = {}
        self._lock = threading.Lock()
        self._next = 0
        self._cb = DONE_FN(self._on_done)

    def _on_done(self, user, status):
        with self._lock:
            fut, keep = self._keep.pop(user)
        if status == OK:
            fut.set_result(keep[-1])
        else:
            fut.set_exception(CafxgError(status, f"{self.kernel} request failed"))

    def request(self, inputs, out: np.ndarray) -> Future:
        """Enqueues one request; `inputs` are numpy arrays (or ctypes arrays),
        `out` receives the reply. Returns a Future resolving to `out`."""
        n = len(inputs)
        ptrs = (C.c_void_p * n)()
        sizes = (C.c_size_t * n)()
        for k, a in enumerate(inputs):
            if isinstance(a, np.ndarray):
                ptrs[k], sizes[k] = a.ctypes.data, a.nbytes
            else:
                ptrs[k], sizes[k] = C.addressof(a), C.sizeof(a)
        fut: Future = Future()
        with self._lock:
            self._next += 1
            token = self._next
            self._keep[token] = (fut, (inputs, ptrs, sizes, out))
        code = lib().cafxg_actor_enqueue(self.handle, ptrs, sizes, n, out.ctypes.data,
                                         out.nbytes, self._cb, token)
        if code != OK:
            with self._lock:
                self._keep.pop(token, None)
            raise CafxgError(code, f"enqueue: {last_error()}")
        return fut

    def reply_bytes(self, inputs) -> int:
        n = len(inputs)
        ptrs = (C.c_void_p * n)()
        sizes = (C.c_size_t * n)()
        for k, a in enumerate(inputs):
            if isinstance(a, np.ndarray):
                ptrs[k], sizes[k] = a.ctypes.data, a.nbytes
            else:
                ptrs[k], sizes[k] = C.addressof(a), C.sizeof(a)
        return lib().cafxg_actor_reply_bytes(self.handle, ptrs, sizes, n)

    def quit(self) -> None:
        _check(lib().cafxg_actor_quit(self.handle), "actor_quit")

    def release(self) -> None:
        if self.handle:
            lib().cafxg_actor_release(self.handle)
            self.handle = None


class Context:
    """A cafxg context over the devices in `device_mask` (0 = all)."""

    def __init__(self, device_mask: int = 0):
        h = C.c_void_p()
        _check(lib().cafxg_open(device_mask, C.byref(h)), "cafxg_open")
        self.handle = h.value
        self._pinned = {}
        # async submits: what a pending submit needs alive (descriptor array,
        # output array, callback), keyed by a token popped when it completes;
        # one CFUNCTYPE object serves every submit and lives with the context
        self._sub_keep = {}
        self._sub_lock = threading.Lock()
        self._sub_next = 0
        self._sub_cb = DONE_FN(self._sub_done)

    def _sub_done(self, user, status):
        with self._sub_lock:
            done, _ = self._sub_keep.pop(user)
        done(status)

    # -- lifetime
    def close(self) -> None:
        if self.handle:
            lib().cafxg_close(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def device_count(self) -> int:
        return lib().cafxg_device_count(self.handle)

    def status(self) -> int:
        """OK, or E_DOWN once a sticky device error made the context unusable."""
        return lib().cafxg_ctx_status(self.handle)

    def sync(self) -> None:
        _check(lib().cafxg_sync(self.handle), "cafxg_sync")

    def stats(self) -> Stats:
        s = Stats()
        _check(lib().cafxg_get_stats(self.handle, C.byref(s)), "get_stats")
        return s

    # -- pinned memory
    def pinned_empty(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        n = int(np.prod(shape)) * dtype.itemsize
        p = C.c_void_p()
        _check(lib().cafxg_host_alloc(self.handle, max(n, 1), C.byref(p)), "host_alloc")
        buf = (C.c_uint8 * max(n, 1)).from_address(p.value)
        arr = np.frombuffer(buf, dtype=np.uint8, count=n).view(dtype).reshape(shape)
        self._pinned[arr.ctypes.data] = p.value
        return arr

    def pinned_free(self, arr: np.ndarray) -> None:
        p = self._pinned.pop(arr.ctypes.data, None)
        if p is not None:
            _check(lib().cafxg_host_free(self.handle, p), "host_free")

    def host_register(self, arr: np.ndarray) -> None:
        _check(lib().cafxg_host_register(self.handle, arr.ctypes.data, arr.nbytes),
               "host_register")

    def host_unregister(self, arr: np.ndarray) -> None:
        _check(lib().cafxg_host_unregister(self.handle, arr.ctypes.data), "host_unregister")

    # -- Mandelbrot
    def mandelbrot(self, tiles, out: np.ndarray | None = None) -> np.ndarray:
        arr, n = _desc_array(tiles)
        if out is None:
            out = np.empty(max(tile_pixels(tiles), 1), dtype=np.uint32)
        _check(lib().cafxg_mandelbrot(self.handle, arr, n, out.ctypes.data), "mandelbrot")
        return out

    def mandelbrot_submit(self, tiles, out: np.ndarray, done) -> None:
        """`done(status)` runs on a backend completion thread."""
        arr, n = _desc_array(tiles)
        with self._sub_lock:
            self._sub_next += 1
            token = self._sub_next
            self._sub_keep[token] = (done, (arr, out))
        code = lib().cafxg_mandelbrot_submit(self.handle, arr, n, out.ctypes.data,
                                             self._sub_cb, token)
        if code != OK:
            with self._sub_lock:
                self._sub_keep.pop(token, None)
        _check(code, "mandelbrot_submit")

    def pending_submits(self) -> int:
        """Async submits whose callback has not run yet."""
        with self._sub_lock:
            return len(self._sub_keep)

    def mandelbrot_device(self, tiles, dev_ptr: int, stream: int = 0, device: int = 0) -> None:
        arr, n = _desc_array(tiles)
        _check(lib().cafxg_mandelbrot_device(self.handle, device, arr, n, dev_ptr,
                                             stream or None), "mandelbrot_device")

    def fnv1a_u32_device(self, dev_ptr: int, n: int, seed: int = 0xCBF29CE484222325,
                         stream: int = 0, device: int = 0) -> int:
        h = C.c_uint64()
        _check(lib().cafxg_fnv1a_u32_device(self.handle, device, dev_ptr, n, seed, C.byref(h),
                                            stream or None), "fnv1a_u32_device")
        return h.value

    def run_mandelbrot(self, size: int, max_iter: int):
        """(checksum, wall_ms) of the reference's run_mandelbrot(size, max_iter)."""
        h, ms = C.c_uint64(), C.c_double()
        _check(lib().cafxg_run_mandelbrot(self.handle, size, max_iter, C.byref(h), C.byref(ms)),
               "run_mandelbrot")
        return h.value, ms.value

    # -- sgemm
    def sgemm(self, A: np.ndarray, B: np.ndarray, C_: np.ndarray | None = None,
              mode: int = SGEMM_AUTO, splits: int = 0) -> np.ndarray:
        M, K = A.shape
        K2, N = B.shape
        assert K == K2
        if C_ is None:
            C_ = np.empty((M, N), dtype=np.float32)
        d = SgemmDesc(M, N, K, A.strides[0] // 4, B.strides[0] // 4, C_.strides[0] // 4, mode,
                      splits)
        _check(lib().cafxg_sgemm(self.handle, C.byref(d), A.ctypes.data, B.ctypes.data,
                                 C_.ctypes.data), "sgemm")
        return C_

    def sgemm_device(self, M, N, K, dA, dB, dC, stream=0, mode=SGEMM_AUTO, device=0,
                     lda=0, ldb=0, ldc=0, splits=0) -> None:
        d = SgemmDesc(M, N, K, lda, ldb, ldc, mode, splits)
        _check(lib().cafxg_sgemm_device(self.handle, device, C.byref(d), dA, dB, dC,
                                        stream or None), "sgemm_device")

    # -- spawn_cl facade
    def spawn(self, kernel: str, dims=(), signature: str | None = None,
              tuning: Tuning | None = None) -> ComputeActor:
        """spawn_cl: `signature` (e.g. "f32*(f32*,f32*)") is checked against
        the kernel's; `tuning` holds launch-shape hints for its requests."""
        n = len(dims)
        d = (C.c_uint64 * max(n, 1))(*dims)
        h = C.c_void_p()
        _check(lib().cafxg_spawn_ex(self.handle, kernel.encode(),
                                    signature.encode() if signature else None, d, n,
                                    C.byref(tuning) if tuning is not None else None,
                                    C.byref(h)), "spawn")
        return ComputeActor(self, h.value, kernel)
