/*
 * cafxg.h -- C ABI of the B200 compute-actor backend (libcafxg.so).
 *
 * This is the drop-in boundary for CAF's GPGPU compute-actor path
 * (`spawn_cl`). The reference runtime's seam
 * is `abstract_actor::enqueue` (/root/reference/proj/include/cafx/
 * abstract_actor.hpp:36); an adapter actor (include/cafxg/gpu_actor.hpp) sits
 * on that seam and forwards each request envelope to the functions below. See
 * INTEGRATION.md for the adapter and the ctypes stub.
 *
 * Rules of the ABI:
 *   - plain C types only; no C++ exception ever crosses it;
 *   - every function is thread-safe; the *_submit and cafxg_actor_enqueue
 *     calls never block on the device (they may block briefly on a host lock);
 *   - status codes are the numeric values of cafx::errc
 *     (/root/reference/proj/include/cafx/error.hpp:11-29), 0 = OK;
 *   - completion callbacks run on a backend-owned completion thread, never on
 *     the caller's thread and never on a cafx scheduler worker. They may call
 *     cafx `deliver`/`enqueue`; they must not call a blocking cafxg function.
 */
#ifndef CAFXG_H
#define CAFXG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAFXG_ABI_VERSION 3  /* 2: cafxg_stats grew nccl_collectives, devices_used;
                                3: peer_gemms */

/* ---- status codes: numeric values of cafx::errc (error.hpp:11-29) --------- */
enum {
  CAFXG_OK = 0,                   /* errc::none */
  CAFXG_E_UNKNOWN_TYPE = 2,       /* errc::unknown_type: unknown kernel name */
  CAFXG_E_OUT_OF_RANGE = 4,       /* errc::out_of_range: bad sizes / offsets */
  CAFXG_E_TYPE_MISMATCH = 5,      /* errc::type_mismatch: wrong buffer bytes */
  CAFXG_E_INTERFACE_MISMATCH = 6, /* errc::interface_mismatch: wrong arity */
  CAFXG_E_CONFIG = 8,             /* errc::config_error: bad argument / state */
  CAFXG_E_SPAWN = 9,              /* errc::spawn_error: no device / init fail */
  CAFXG_E_TIMEOUT = 13,           /* errc::request_timeout */
  CAFXG_E_DOWN = 14               /* errc::request_down: actor or device gone */
};

typedef struct cafxg_ctx cafxg_ctx;
typedef struct cafxg_actor cafxg_actor;

/* Completion callback: `status` is a CAFXG_* code. Runs on a completion
 * thread owned by the context. */
typedef void (*cafxg_done_fn)(void* user, int status);

int cafxg_abi_version(void);
/* Static description of a status code. */
const char* cafxg_status_string(int status);
/* Context string of the last failure on the calling thread ("" if none). */
const char* cafxg_last_error(void);

/* ---- context --------------------------------------------------------------
 * device_mask: bit i selects visible CUDA device i; 0 selects every visible
 * device. Opening creates per-device streams, pools, dispatcher and completion
 * threads (and, with >1 device, the NCCL communicator, loaded lazily). */
int cafxg_open(uint64_t device_mask, cafxg_ctx** out);
/* Drains in-flight work, fails queued actor requests with CAFXG_E_DOWN and
 * releases everything. */
int cafxg_close(cafxg_ctx* ctx);
int cafxg_device_count(const cafxg_ctx* ctx);
/* CAFXG_OK while the context is usable; CAFXG_E_DOWN after a sticky device
 * error (illegal address, launch failure, ECC, ...: the CUDA context is
 * gone), with the cause in cafxg_last_error(). From then on every submission
 * fails with CAFXG_E_DOWN; an adapter should terminate its compute actors
 * (monitors and pending requesters fire, abstract_actor.cpp:108-134). */
int cafxg_ctx_status(cafxg_ctx* ctx);
/* Blocks until every submission made before the call has completed and its
 * callback has returned. */
int cafxg_sync(cafxg_ctx* ctx);

/* ---- pinned host memory ----------------------------------------------------
 * Page-locked, device-mapped buffers from a per-context pool. Request and
 * reply buffers that live here are moved by DMA / written by kernels directly
 * (no staging copy); any other host pointer is staged through the pool. */
int cafxg_host_alloc(cafxg_ctx* ctx, size_t bytes, void** ptr);
int cafxg_host_free(cafxg_ctx* ctx, void* ptr);
/* Page-locks and maps caller memory (e.g. a shared-memory image several
 * ranks gather into) so replies land there by DMA without staging. */
int cafxg_host_register(cafxg_ctx* ctx, void* ptr, size_t bytes);
int cafxg_host_unregister(cafxg_ctx* ctx, void* ptr);

/* ---- Mandelbrot -------------------------------------------------------------
 * Generalised escape-time request. Pixel (col,row)
 * of a width x height image over [x0,x1] x [y0,y1] samples
 *     cr = x0 + ((col + s) * (x1 - x0)) / width,
 *     ci = y0 + ((row + s) * (y1 - y0)) / height       (fp64, IEEE, no FMA)
 * with s = 0 (CAFXG_CORNER) or 0.5 (CAFXG_CENTRE), rounded to binary32 for
 * CAFXG_FP32. The count is the reference's mandelbrot_cell
 * (bench.cpp:367-379) evaluated op-for-op in the chosen precision. Row 0 is
 * y0. Reference mode (x0=-1.5,x1=0.5,y0=-1,y1=1, corner, fp64, W=H=size)
 * reproduces run_mandelbrot's cells bit for bit.
 *
 * A tile covers rows [row0,row0+nrows) x cols [col0,col0+ncols); its counts
 * are written row-major with pitch ncols starting at element `out_offset` of
 * the output buffer. */
enum { CAFXG_FP32 = 0, CAFXG_FP64 = 1 };
enum { CAFXG_CORNER = 0, CAFXG_CENTRE = 1 };

typedef struct {
  double x0, x1, y0, y1;
  uint32_t width, height;
  uint32_t row0, nrows;
  uint32_t col0, ncols;
  uint32_t max_iter;
  uint32_t precision; /* CAFXG_FP32 | CAFXG_FP64 */
  uint32_t sampling;  /* CAFXG_CORNER | CAFXG_CENTRE */
  uint32_t reserved;
  uint64_t out_offset; /* in uint32 elements */
} cafxg_mandel_desc;

/* Host-to-host request: all `n` tiles of one batch in one launch per device,
 * counts written into `host_out`. Non-blocking; `done` (may be NULL) fires on
 * the completion thread. With >1 device the tiles' rows are dealt to the
 * devices in cyclic chunks. */
int cafxg_mandelbrot_submit(cafxg_ctx* ctx, const cafxg_mandel_desc* tiles,
                            size_t n, uint32_t* host_out, cafxg_done_fn done,
                            void* user);
/* Blocking convenience wrapper around cafxg_mandelbrot_submit. */
int cafxg_mandelbrot(cafxg_ctx* ctx, const cafxg_mandel_desc* tiles, size_t n,
                     uint32_t* host_out);
/* Device-resident launch: counts go to device memory `dev_out` on context
 * device `device`, on `stream` (a cudaStream_t; NULL = the context's compute
 * stream for that device). Only enqueues work. */
int cafxg_mandelbrot_device(cafxg_ctx* ctx, int device,
                            const cafxg_mandel_desc* tiles, size_t n,
                            uint32_t* dev_out, void* stream);

/* FNV-1a-64 of `n` device-resident u32 cells hashed as big-endian bytes
 * (cafx::detail::fnv1a_u32, fnv.hpp:23-28) starting from `seed`; blocks until
 * the hash is in *hash. Parallelised through the low-byte/affine decomposition
 * of the FNV state; bit-identical to the serial loop. */
int cafxg_fnv1a_u32_device(cafxg_ctx* ctx, int device, const uint32_t* cells,
                           uint64_t n, uint64_t seed, uint64_t* hash,
                           void* stream);
/* The reference's run_mandelbrot(size, max_iter) (bench.cpp:481-505): the
 * fp64 reference-mode image over [-1.5,0.5]x[-1,1] computed on the context's
 * devices and its collector checksum (bench.cpp:329-331) computed on device.
 * Blocking; *wall_ms (may be NULL) is request-to-checksum wall clock. */
int cafxg_run_mandelbrot(cafxg_ctx* ctx, uint32_t size, uint32_t max_iter,
                         uint64_t* checksum, double* wall_ms);

/* ---- fp32 matrix multiply --------------------------------------------------
 * C = A * B, row-major, the OpenCL `matrix_multiply(matrix1, matrix2, output)`
 * contract. */
/* The 3xTF32 path takes M % 128 == 0, N % 128 == 0, K % 32 == 0 (M, N >= 128),
 * lda, ldc multiples of 4 and, for device-resident calls, A and C 16-byte
 * aligned; AUTO runs the FFMA kernel otherwise and 3XTF32 fails with
 * CAFXG_E_CONFIG. Results are within 1e-5 normwise of an fp64-accumulated
 * product either way. */
enum {
  CAFXG_SGEMM_AUTO = 0,   /* 3xTF32 tensor cores when shapes allow, else FFMA */
  CAFXG_SGEMM_FFMA = 1,   /* register-tiled SIMT fp32 FFMA */
  CAFXG_SGEMM_3XTF32 = 2  /* tcgen05 kind::tf32, big*big + big*small + small*big */
};

typedef struct {
  uint32_t M, N, K;
  uint32_t lda, ldb, ldc; /* 0 = packed (K, N, N) */
  uint32_t mode;          /* CAFXG_SGEMM_* */
  uint32_t splits;        /* 3xTF32 split-K cluster size 1/2/4/8; 0 = chosen per shape */
} cafxg_sgemm_desc;

/* Host-to-host request. With >1 device, A is split into row blocks per
 * device and B is replicated (H2D of 1/G of B per device + NCCL all-gather
 * over NVLink). Non-blocking. */
int cafxg_sgemm_submit(cafxg_ctx* ctx, const cafxg_sgemm_desc* d,
                       const float* A, const float* B, float* C,
                       cafxg_done_fn done, void* user);
int cafxg_sgemm(cafxg_ctx* ctx, const cafxg_sgemm_desc* d, const float* A,
                const float* B, float* C);
/* Device-resident launch on context device `device` (pointers are device
 * memory on that device). Scratch for the 3xTF32 split comes from the
 * context's device pool. */
int cafxg_sgemm_device(cafxg_ctx* ctx, int device, const cafxg_sgemm_desc* d,
                       const float* A, const float* B, float* C, void* stream);

/* ---- spawn_cl facade: compute actors ---------------------------------------
 * cafxg_spawn is `spawn_cl<Out(In...)>(source, kernel_name, dims)` with the
 * OpenCL source replaced by a precompiled sm_100a kernel looked up by name:
 *   "mandelbrot"      dims = {} ; request inputs: 1 buffer holding one or
 *                     more cafxg_mandel_desc ; output: uint32 counts
 *                     (sum of tile pixels, tiles packed in order; out_offset
 *                     is ignored and recomputed).
 *   "matrix_multiply" dims = {size, size} ; inputs: matrix1,
 *                     matrix2 (size*size floats each) ; output size*size
 *                     floats.
 * The actor owns an MPSC mailbox; a per-device dispatcher drains every
 * actor's mailbox, batches compatible requests into one launch (one grid over
 * all queued tiles), and a completion thread fires each request's callback
 * (the cafx adapter turns that into the reply envelope,
 * local_actor.cpp:319-329). */
int cafxg_spawn(cafxg_ctx* ctx, const char* kernel_name, const uint64_t* dims,
                size_t ndims, cafxg_actor** out);

/* The kernel's signature normalised the way spawn_cl takes it (PAPER.md:
 * 357-361: a result type instead of the trailing output parameter), as text:
 *   "matrix_multiply" -> "f32*(f32*,f32*)"    spawn_cl<float*(float*,float*)>
 *   "mandelbrot"      -> "u32*(mandel_desc*)" spawn_cl<uint32_t*(cafxg_mandel_desc*)>
 * (f32 = float, u32 = uint32_t, mandel_desc = cafxg_mandel_desc). Writes it
 * NUL-terminated into buf (cap bytes); CAFXG_E_UNKNOWN_TYPE for unknown
 * kernels, CAFXG_E_OUT_OF_RANGE if cap is too small. */
int cafxg_kernel_signature(const char* kernel_name, char* buf, size_t cap);

/* spawn_cl's tuning overload: launch-shape hints stored with the actor and
 * applied to every request it serves (the OpenCL nd_range / work-group
 * arguments have no meaning for these kernels; these are their knobs).
 * Zero fields keep the backend's choice. */
typedef struct {
  uint32_t block_steps;  /* mandelbrot: escape-test interval of the deferred
                            kernel, 16..64 and a multiple of 8 (steps run
                            unchecked between tests); 0 = cost model */
  uint32_t max_ctas;     /* mandelbrot: cap on the CTAs of a launch (shares
                            the GPU with other work); 0 = every SM at full
                            occupancy */
  uint32_t sgemm_mode;   /* matrix_multiply: CAFXG_SGEMM_* */
  uint32_t sgemm_splits; /* matrix_multiply: split-K cluster size 1/2/4/8 */
  uint32_t reserved[4];  /* must be 0 */
} cafxg_tuning;

/* cafxg_spawn with the spawn_cl template signature checked against the
 * kernel's (`signature` may be NULL: unchecked; a mismatch fails with
 * CAFXG_E_INTERFACE_MISMATCH before any actor exists) and optional tuning
 * (NULL = defaults; out-of-range values fail with CAFXG_E_CONFIG). */
int cafxg_spawn_ex(cafxg_ctx* ctx, const char* kernel_name, const char* signature,
                   const uint64_t* dims, size_t ndims, const cafxg_tuning* tuning,
                   cafxg_actor** out);
/* Enqueues one request. in[i]/in_bytes[i] are the request's input buffers;
 * the reply is written to out/out_bytes before `done(user, status)` runs.
 * Buffers must stay valid until then. Size checks happen here (returning the
 * error synchronously) so a malformed request never reaches the device. */
int cafxg_actor_enqueue(cafxg_actor* a, const void* const* in,
                        const size_t* in_bytes, size_t n_in, void* out,
                        size_t out_bytes, cafxg_done_fn done, void* user);
/* Expected reply size in bytes for the given inputs (0 on error). */
size_t cafxg_actor_reply_bytes(cafxg_actor* a, const void* const* in,
                               const size_t* in_bytes, size_t n_in);
/* Inside a done callback of cafxg_actor_enqueue: how many request completions
 * the backend is delivering together with this one on this thread (the
 * requests of one launch), 1 for a lone reply. Lets an adapter batch the
 * delivery of many replies and hand a lone one over at once. */
size_t cafxg_completion_batch(void);
/* Terminates the actor: queued (not yet launched) requests complete with
 * CAFXG_E_DOWN, launched ones finish normally; later enqueues fail with
 * CAFXG_E_DOWN. Mirrors the hard-kill exit path (actor_system.cpp:243-258). */
int cafxg_actor_quit(cafxg_actor* a);
/* Drops the caller's reference (quits first if still alive). */
int cafxg_actor_release(cafxg_actor* a);

/* ---- statistics --------------------------------------------------------- */
typedef struct {
  uint64_t requests;       /* actor requests completed */
  uint64_t batches;        /* dispatcher batches (one launch each) */
  uint64_t kernel_launches;/* kernels launched by the backend */
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t max_batch;      /* largest batch seen */
  uint64_t direct_batches; /* batches whose escape kernel wrote the replies itself */
  uint64_t nccl_collectives; /* NCCL collectives issued (multi-device B all-gather) */
  uint64_t devices_used;   /* bit i set: context device i has run a kernel */
  uint64_t peer_gemms;     /* multi-device GEMMs that read B's slices from the peers in place */
} cafxg_stats;
int cafxg_get_stats(cafxg_ctx* ctx, cafxg_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* CAFXG_H */
