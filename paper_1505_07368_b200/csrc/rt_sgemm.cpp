// libcafxg.so host runtime, fp32 matrix multiply: device launches, the
// host row-block pipeline, the 2D wavefront for large requests and the
// multi-device split with B replicated over NCCL (or peer copies).
#include "runtime_internal.hpp"

namespace cafxg {

// ---- sgemm ---------------------------------------------------------------------------

int validate_sgemm(cafxg_sgemm_desc& d) {
  if (d.lda == 0) d.lda = d.K;
  if (d.ldb == 0) d.ldb = d.N;
  if (d.ldc == 0) d.ldc = d.N;
  if (d.lda < d.K || d.ldb < d.N || d.ldc < d.N)
    return fail(CAFXG_E_OUT_OF_RANGE, "sgemm: leading dimension below extent");
  if (d.mode > CAFXG_SGEMM_3XTF32)
    return fail(CAFXG_E_CONFIG, "sgemm: bad mode");
  if (d.splits > 8 || (d.splits & (d.splits - 1)))
    return fail(CAFXG_E_CONFIG, "sgemm: splits must be 0, 1, 2, 4 or 8");
  if (d.M > (1u << 30) || d.N > (1u << 30) || d.K > (1u << 30))
    return fail(CAFXG_E_OUT_OF_RANGE, "sgemm: dimension too large");
  return CAFXG_OK;
}

// Runs C = A*B on one device with device pointers.
int sgemm_on_device(cafxg_ctx* ctx, Device* d, const cafxg_sgemm_desc& g,
                           const float* A, const float* B, float* C,
                           cudaStream_t stream) {
  if (g.M == 0 || g.N == 0)
    return CAFXG_OK;
  if (g.K == 0) {
    for (uint32_t r = 0; r < g.M; ++r)
      CAFXG_CUDA_TRY(cudaMemsetAsync(C + (size_t)r * g.ldc, 0, g.N * 4, stream));
    return CAFXG_OK;
  }
  // AUTO takes the 3xTF32 tensor-core path for supported shapes (validated:
  // <= 1.4e-6 normwise up to 16384^3); CAFXG_SGEMM_AUTO_TC=0
  // forces the FFMA kernel.
  static const bool auto_tc = [] {
    const char* e = getenv("CAFXG_SGEMM_AUTO_TC");
    return !(e && e[0] == '0');
  }();
  // the tensor-core path reads A and writes C in 16-byte vectors (device-API
  // callers pass arbitrary pointers; host requests use the pool's buffers)
  const bool aligned = ((uintptr_t)A & 15) == 0 && ((uintptr_t)C & 15) == 0;
  bool supported = aligned && sgemm_tc_supported(g.M, g.N, g.K, g.lda, g.ldb, g.ldc);
  bool tc = supported && (g.mode == CAFXG_SGEMM_3XTF32 || (g.mode == CAFXG_SGEMM_AUTO && auto_tc));
  if (g.mode == CAFXG_SGEMM_3XTF32 && !tc)
    return fail(CAFXG_E_CONFIG,
                "sgemm: shape or alignment not supported by the 3xTF32 kernel (see cafxg.h)");
  if (tc) {
    size_t sb = sgemm_tc_scratch_bytes(g.M, g.N, g.K, d->sms, (int)g.splits);
    void* scratch = nullptr;
    CAFXG_CUDA_TRY(cudaMallocAsync(&scratch, sb, stream));
    int launches = 0;
    int e = sgemm_tc_launch(A, B, C, g.M, g.N, g.K, g.lda, g.ldb, g.ldc, scratch,
                            d->sms, stream, &launches, (int)g.splits);
    ctx->st_launches += launches;
    mark_used(ctx, d);
    CAFXG_CUDA_TRY(cudaFreeAsync(scratch, stream));
    if (e != 0)
      return cuda_status((cudaError_t)e, "sgemm 3xtf32 launch");
    return CAFXG_OK;
  }
  int e = sgemm_simt_launch(A, B, C, g.M, g.N, g.K, g.lda, g.ldb, g.ldc, stream);
  if (e != 0)
    return cuda_status((cudaError_t)e, "sgemm simt launch");
  ctx->st_launches++;
  mark_used(ctx, d);
  return CAFXG_OK;
}

static bool nccl_selftest() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_NCCL_SELFTEST");
    return e && e[0] == '1';
  }();
  return on;
}

int ensure_nccl(cafxg_ctx* ctx) {
  std::lock_guard<std::mutex> g(ctx->nccl_mu);
  if (!ctx->comms.empty())
    return CAFXG_OK;
  if (ctx->virtual_devs)
    return fail(CAFXG_E_CONFIG, "virtual devices share one GPU; NCCL not used");
  if (ctx->nccl_failed)
    return fail(CAFXG_E_SPAWN, "NCCL unavailable (first attempt failed)");
  ctx->nccl_failed = true;  // cleared on success
  if (!ctx->nccl.load())
    return fail(CAFXG_E_SPAWN, "libnccl.so.2 not loadable");
  std::vector<int> ords;
  for (auto& d : ctx->devs)
    ords.push_back(d->ordinal);
  std::vector<ncclComm_t> comms(ords.size());
  ncclResult_t r = ctx->nccl.CommInitAll(comms.data(), (int)ords.size(), ords.data());
  if (r != ncclSuccess)
    return fail(CAFXG_E_SPAWN, "ncclCommInitAll failed: %s",
                ctx->nccl.GetErrorString ? ctx->nccl.GetErrorString(r) : "?");
  ctx->comms = comms;
  ctx->nccl_failed = false;
  return CAFXG_OK;
}

// ---- multi-device GEMM fused with the exchange of B ----------------------------
// B is uploaded in K slices, 1/G per device (each device also makes the lo
// halves of its slice); every device then multiplies its row block of A by
// the whole of B with sgemm_tc_peer_gemm, whose TMA loads read each k-block
// from the device that holds its slice -- over NVLink for the peers' slices.
// The all-gather of the NCCL path disappears into the GEMM: remote tiles are
// fetched as the tensor cores consume them, overlapped with the MMAs of the
// earlier stages, and no device holds a full copy of B. Needs peer access
// between every pair of the context's GPUs (virtual devices share one GPU,
// where the "peer" slices are local: the same code path, tested on one GPU).
// CAFXG_SGEMM_P2P=0 at cafxg_open keeps that context on the NCCL all-gather
// path (read per context, so one process can compare both exchanges).

static bool peer_access_all(cafxg_ctx* ctx) {
  std::lock_guard<std::mutex> g(ctx->nccl_mu);  // (serialises the one-time enabling)
  if (ctx->p2p_state)
    return ctx->p2p_state > 0;
  int ok = 1;
  for (auto& a : ctx->devs)
    for (auto& b : ctx->devs) {
      if (a->ordinal == b->ordinal)
        continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, a->ordinal, b->ordinal) != cudaSuccess || !can) {
        ok = -1;
        continue;
      }
      cudaSetDevice(a->ordinal);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b->ordinal, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        ok = -1;
      // The slices of B come from b's stream-ordered pool (cudaMallocAsync),
      // which cudaDeviceEnablePeerAccess does not cover: the pool itself
      // must map its allocations for a, or a's TMA loads of them fault.
      cudaMemPool_t pool;
      cudaMemAccessDesc acc = {};
      acc.location.type = cudaMemLocationTypeDevice;
      acc.location.id = a->ordinal;
      acc.flags = cudaMemAccessFlagsProtReadWrite;
      if (cudaDeviceGetDefaultMemPool(&pool, b->ordinal) != cudaSuccess ||
          cudaMemPoolSetAccess(pool, &acc, 1) != cudaSuccess)
        ok = -1;
    }
  cudaGetLastError();
  ctx->p2p_state = ok;
  return ok > 0;
}

static bool p2p_eligible(cafxg_ctx* ctx, const cafxg_sgemm_desc& g, uint32_t rows_per) {
  const int G = (int)ctx->devs.size();
  return G > 1 && !ctx->p2p_off && g.mode != CAFXG_SGEMM_FFMA && g.K % G == 0 &&
         g.M % 128 == 0 && rows_per % 128 == 0 && sgemm_tc_peer_supported(128, g.N, g.K, G) &&
         peer_access_all(ctx);
}

static int sgemm_p2p_submit(cafxg_ctx* ctx, const cafxg_sgemm_desc& g, const float* A,
                            const float* B, float* C, uint32_t rows_per, Join* join) {
  const size_t G = ctx->devs.size(), M = g.M, N = g.N, K = g.K, ks = K / G;
  std::vector<std::unique_lock<std::mutex>> locks;
  for (auto& d : ctx->devs)
    locks.emplace_back(d->submit_mu);
  int status = CAFXG_OK;
  auto note = [&](int s) {
    if (status == CAFXG_OK && s != CAFXG_OK)
      status = s;
  };
  std::vector<float*> dB(G, nullptr), dBl(G, nullptr), dA(G, nullptr), dAl(G, nullptr),
      dC(G, nullptr);
  std::vector<cudaEvent_t> ready(G, nullptr), done(G, nullptr);
  std::vector<std::vector<cudaEvent_t>> held(G);  // per device: events back to its pool
  auto ev = [&](size_t k, cudaStream_t sm) {
    cudaEvent_t e = pooled_event(ctx->devs[k].get());
    if (e) {
      cudaEventRecord(e, sm);
      held[k].push_back(e);
    }
    return e;
  };
  auto rows_of = [&](size_t k) {
    const size_t r0 = std::min<size_t>(M, rows_per * k), r1 = std::min<size_t>(M, rows_per * (k + 1));
    return std::make_pair(r0, r1 - r0);
  };
  // A row blocks per device (whole 128-row tiles): uploads, GEMMs and
  // downloads of consecutive blocks overlap on the three streams. Every
  // block's GEMM streams all of B again (its K slices, 7/8 of them over
  // NVLink at 8 GPUs), so blocks keep >= 1024 rows: each block then does
  // >= 6 x 1024 tensor flops (3 MMAs) per 8 bytes of B it streams (quarter
  // blocks of cfg5's 2048 rows per device at 8 GPUs would read B 4x over).
  // CAFXG_P2P_RMIN overrides the minimum (tests: several blocks on small
  // shapes).
  static const size_t rmin = [] {
    const char* e = getenv("CAFXG_P2P_RMIN");
    const long v = e ? atol(e) : 0;
    return v > 0 ? (size_t)(v + 127) / 128 * 128 : (size_t)1024;
  }();
  auto blocks_of = [](size_t m) {
    std::vector<size_t> b;
    const size_t R = std::max<size_t>(rmin, (m / 4 + 127) / 128 * 128);
    for (size_t r = 0; r < m; r += R)
      b.push_back(std::min(R, m - r));
    return b;
  };
  // 1. each device: buffers; its K slice of B up on the upload stream, then
  // the slice's lo halves; its A row blocks up behind the slice
  std::vector<std::vector<cudaEvent_t>> a_up(G);
  for (size_t k = 0; k < G; ++k) {
    Device* d = ctx->devs[k].get();
    cudaSetDevice(d->ordinal);
    cudaStream_t cs = d->compute;
    const size_t m = rows_of(k).second;
    if (status == CAFXG_OK &&
        (cudaMallocAsync((void**)&dB[k], ks * N * 4, cs) != cudaSuccess ||
         cudaMallocAsync((void**)&dBl[k], ks * N * 4, cs) != cudaSuccess ||
         (m && (cudaMallocAsync((void**)&dA[k], m * K * 4, cs) != cudaSuccess ||
                cudaMallocAsync((void**)&dAl[k], m * K * 4, cs) != cudaSuccess ||
                cudaMallocAsync((void**)&dC[k], m * N * 4, cs) != cudaSuccess))))
      note(cuda_status(cudaGetLastError(), "sgemm p2p: allocation"));
    if (status == CAFXG_OK)
      note(stream_after_pooled(d, d->h2d, cs));
    if (status == CAFXG_OK) {
      note(cuda_status(cudaMemcpy2DAsync(dB[k], N * 4, B + k * ks * g.ldb, (size_t)g.ldb * 4,
                                         N * 4, ks, cudaMemcpyHostToDevice, d->h2d),
                       "sgemm p2p: B slice upload"));
      ctx->st_h2d += ks * N * 4;
    }
    cudaEvent_t b_up = status == CAFXG_OK ? ev(k, d->h2d) : nullptr;
    size_t r = rows_of(k).first;
    for (size_t mb : blocks_of(m)) {
      if (status != CAFXG_OK)
        break;
      note(cuda_status(cudaMemcpy2DAsync(dA[k] + (r - rows_of(k).first) * K, K * 4,
                                         A + r * g.lda, (size_t)g.lda * 4, K * 4, mb,
                                         cudaMemcpyHostToDevice, d->h2d),
                       "sgemm p2p: A upload"));
      ctx->st_h2d += mb * K * 4;
      a_up[k].push_back(ev(k, d->h2d));
      r += mb;
    }
    if (status == CAFXG_OK) {
      if (b_up)
        cudaStreamWaitEvent(cs, b_up, 0);
      const int e = sgemm_tc_lo(dB[k], (int)N, (int)ks, (int)N, dBl[k], d->sms, cs);
      note(e ? cuda_status((cudaError_t)e, "sgemm p2p: B lo pass") : CAFXG_OK);
      ctx->st_launches++;
    }
    ready[k] = ev(k, cs);
  }
  // 2. each device: its A row blocks times all of B (peer slices read in
  // place), each block's C down as soon as its GEMM is done
  for (size_t k = 0; k < G; ++k) {
    Device* d = ctx->devs[k].get();
    cudaSetDevice(d->ordinal);
    cudaStream_t cs = d->compute;
    for (size_t j = 0; j < G; ++j)
      if (ready[j])
        cudaStreamWaitEvent(cs, ready[j], 0);
    const auto [r0, m] = rows_of(k);
    size_t off = 0, bi = 0;
    for (size_t mb : blocks_of(m)) {
      if (status != CAFXG_OK)
        break;
      if (bi < a_up[k].size() && a_up[k][bi])
        cudaStreamWaitEvent(cs, a_up[k][bi], 0);
      int e = sgemm_tc_lo(dA[k] + off * K, (int)K, (int)mb, (int)K, dAl[k] + off * K, d->sms,
                          cs);
      if (!e)
        e = sgemm_tc_peer_gemm(dA[k] + off * K, (int)K, dAl[k] + off * K, (int)mb, (int)N,
                               (int)K, dB.data(), dBl.data(), (int)G, dC[k] + off * N, (int)N,
                               cs);
      note(e ? cuda_status((cudaError_t)e, "sgemm p2p: GEMM launch") : CAFXG_OK);
      ctx->st_launches += 2;
      mark_used(ctx, d);
      if (cudaEvent_t gdone = ev(k, cs))
        cudaStreamWaitEvent(d->d2h, gdone, 0);
      if (status == CAFXG_OK) {
        note(cuda_status(cudaMemcpy2DAsync(C + (r0 + off) * g.ldc, (size_t)g.ldc * 4,
                                           dC[k] + off * N, N * 4, N * 4, mb,
                                           cudaMemcpyDeviceToHost, d->d2h),
                         "sgemm p2p: C download"));
        ctx->st_d2h += mb * N * 4;
      }
      off += mb;
      ++bi;
    }
    // the part completes on the download stream, behind every kernel and
    // copy of this device (also on failure: queued uploads may still read
    // the caller's A and B, queued downloads write its C)
    stream_after_pooled(d, cs, d->h2d);
    done[k] = ev(k, cs);
    stream_after_pooled(d, d->d2h, cs);
    for (float* p : {dA[k], dAl[k], dC[k]})
      if (p)
        cudaFreeAsync(p, d->d2h);
  }
  // 3. a slice is freed once every device's GEMM has read it; each device's
  // part completes behind that (so behind every device's download)
  for (size_t k = 0; k < G; ++k) {
    Device* d = ctx->devs[k].get();
    cudaSetDevice(d->ordinal);
    for (size_t j = 0; j < G; ++j)
      if (done[j])
        cudaStreamWaitEvent(d->compute, done[j], 0);
    if (dB[k])
      cudaFreeAsync(dB[k], d->compute);
    if (dBl[k])
      cudaFreeAsync(dBl[k], d->compute);
  }
  // every wait on the events is enqueued: back to their pools
  for (size_t k = 0; k < G; ++k) {
    Device* d = ctx->devs[k].get();
    for (cudaEvent_t e : held[k])
      d->ev_pool.push_back(e);
  }
  const int st = status;
  for (size_t k = 0; k < G; ++k) {
    Device* d = ctx->devs[k].get();
    cudaSetDevice(d->ordinal);
    if (st != CAFXG_OK)
      push_completion(ctx, d, d->d2h, [join, st](int) { join->part_done(st); });
    else
      push_completion(ctx, d, d->d2h, [join](int s) { join->part_done(s); });
  }
  return CAFXG_OK;
}

// Host-request pipeline for one device's C rows [r0, r1) with B already in
// device memory (dB, K x N): B is split once (tf32 hi/lo, transposed), then
// per block of R rows: H2D of A_i on the upload stream -> hi/lo split + 3xTF32
// GEMM on the compute stream -> D2H of C_i on the download stream. A and C
// blocks are double-buffered, so PCIe traffic in both directions overlaps the
// tensor-core work. Completion is recorded on d2h.
bool sgemm_pipeline_eligible(const cafxg_sgemm_desc& g, uint32_t rows) {
  return g.mode != CAFXG_SGEMM_FFMA && rows >= 1024 && rows % 128 == 0 &&
         sgemm_tc_supported(128, g.N, g.K, g.K, g.N, g.N);
}

// hostB: when non-null, B (K x N, host) is uploaded here on the upload
// stream, ahead of the A blocks, instead of by the caller into dB: the first A
// block then follows B over PCIe without waiting for B's split.
int sgemm_pipeline_device(cafxg_ctx* ctx, Device* d, const cafxg_sgemm_desc& g,
                                 const float* A, const float* dB, float* C, uint32_t r0,
                                 uint32_t r1, const float* hostB = nullptr) {
  const size_t N = g.N, K = g.K;
  const uint32_t rows = r1 - r0;
  uint32_t R = ((rows + 7) / 8 + 127) / 128 * 128;  // ~8 blocks of whole 128-row tiles
  // minimum block height (CAFXG_SGEMM_RMIN: experiments only): 256 since the
  // GEMM launch follows the split with PDL (e2e 1024^3 0.275 -> 0.272 ms
  // median, 2048^3 0.906 -> 0.869 ms; 128 lost at 1024^3)
  static const uint32_t rmin = [] {
    const char* e = getenv("CAFXG_SGEMM_RMIN");
    return e ? (uint32_t)atoi(e) : 256u;
  }();
  R = std::max<uint32_t>(R, rmin);
  // Raw operands (the device-API size rule): A blocks and B are read as they
  // lie and only their lo halves are made (no transpose of B, half the
  // writes); split-K reduces through an L2 workspace (one more piece).
  // 1024^3 end to end: the four block GEMMs were the critical path (~40 us
  // each through the split + transpose pass and the DSMEM reduction).
  const bool raw = sgemm_tc_raw_wanted((int)rows, (int)N);
  const int bn = sgemm_tc_pick_bn((int)R, (int)N, d->sms);
  const int splits_max = g.splits ? (int)g.splits : sgemm_tc_splits((int)R, (int)N, (int)K, d->sms, bn);
  const size_t ws_bytes = raw ? sgemm_tc_ws_bytes((int)R, (int)N, splits_max, bn) : 0;
  float *Bh = nullptr, *Bl = nullptr, *Ah = nullptr, *Al = nullptr, *wsk = nullptr;
  float* dA[2] = {nullptr, nullptr};
  float* dC[2] = {nullptr, nullptr};
  cudaStream_t cs = d->compute;
  // buffers carved from the device's grow-only workspace (a stream-ordered
  // allocation and free per buffer and request cost more host time than the
  // GEMMs of a 1024^3 request); 256-byte aligned pieces
  {
    const size_t pieces[9] = {N * K, N * K, (size_t)R * K, (size_t)R * K, (size_t)R * K,
                              (size_t)R * K, (size_t)R * N, (size_t)R * N, ws_bytes / 4};
    size_t need = 0;
    for (size_t p : pieces)
      need += (p * 4 + 255) / 256 * 256;
    if (d->sgemm_ws_bytes < need) {
      if (d->sgemm_ws) {
        cudaStreamSynchronize(d->h2d);
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(d->d2h);
        cudaFree(d->sgemm_ws);
        d->sgemm_ws = nullptr;
        d->sgemm_ws_bytes = 0;
      }
      CAFXG_CUDA_TRY(cudaMalloc((void**)&d->sgemm_ws, need));
      d->sgemm_ws_bytes = need;
    }
    float** dst[9] = {&Bh, &Bl, &Ah, &Al, &dA[0], &dA[1], &dC[0], &dC[1], &wsk};
    uint8_t* base = reinterpret_cast<uint8_t*>(d->sgemm_ws);
    for (int i = 0; i < 9; ++i) {
      *dst[i] = reinterpret_cast<float*>(base);
      base += (pieces[i] * 4 + 255) / 256 * 256;
    }
  }
  // the previous request's kernels and downloads are done with the workspace
  // before this one's uploads and kernels touch it
  CAFXG_TRY(stream_after_pooled(d, cs, d->d2h));
  CAFXG_TRY(stream_after_pooled(d, d->h2d, cs));
  // CAFXG_TRACE=1: device timeline of the request (uploads, GEMMs, downloads)
  std::vector<std::pair<const char*, cudaEvent_t>> tev;
  const double t_host0 = trace_now_ms();
  auto tmark = [&](const char* what, cudaStream_t sm) {
    if (!trace_on())
      return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, sm);
    tev.emplace_back(what, e);
  };
  tmark("start", d->h2d);
  if (hostB) {
    CAFXG_CUDA_TRY(cudaMemcpyAsync(const_cast<float*>(dB), hostB, K * N * 4,
                                   cudaMemcpyHostToDevice, d->h2d));
    ctx->st_h2d += K * N * 4;
    tmark("B up", d->h2d);
    CAFXG_TRY(stream_after_pooled(d, cs, d->h2d));
  }
  // tensor maps encoded once per request: every block reuses Ah/Al (R rows)
  // and Bh/Bl; raw: one set per A slot (the maps read the slot itself), Bl
  // holds lo(B) in B's layout, Al lo of the current block
  SgemmTcMaps maps, rmaps[2];
  int e = 0;
  if (raw) {
    e = sgemm_tc_lo(dB, (int)N, (int)K, (int)N, Bl, d->sms, cs);
    for (int sl = 0; sl < 2 && !e; ++sl)
      e = sgemm_tc_make_maps_raw(dA[sl], (int)K, Al, (int)R, dB, (int)N, Bl, (int)N, (int)K, bn,
                                 &rmaps[sl]);
  } else {
    e = sgemm_tc_split_b(dB, (int)N, (int)K, (int)N, Bh, Bl, cs);
    if (!e)
      e = sgemm_tc_make_maps(Ah, Al, (int)R, Bh, Bl, (int)N, (int)K, bn, &maps);
  }
  if (e != 0)
    return cuda_status((cudaError_t)e, "sgemm: B split / tensor maps");
  ctx->st_launches++;
  std::vector<cudaEvent_t> ev_split, ev_gemm, ev_down;
  auto mk = [d](std::vector<cudaEvent_t>& v) {
    cudaEvent_t ev = pooled_event(d);
    v.push_back(ev);
    return ev;
  };
  int status = CAFXG_OK;
  uint32_t i = 0;
  for (uint32_t b0 = 0; b0 < rows && status == CAFXG_OK; b0 += R, ++i) {
    const uint32_t m = std::min(R, rows - b0);
    const int slot = i & 1;
    // upload A block (slot free once block i-2's split -- raw: its GEMM --
    // consumed it)
    if (i >= 2)
      cudaStreamWaitEvent(d->h2d, raw ? ev_gemm[i - 2] : ev_split[i - 2], 0);
    const float* src = A + (size_t)(r0 + b0) * g.lda;
    if (g.lda == K)
      status = cuda_status(cudaMemcpyAsync(dA[slot], src, (size_t)m * K * 4,
                                           cudaMemcpyHostToDevice, d->h2d), "sgemm: A upload");
    else
      status = cuda_status(cudaMemcpy2DAsync(dA[slot], K * 4, src, (size_t)g.lda * 4, K * 4, m,
                                             cudaMemcpyHostToDevice, d->h2d),
                           "sgemm: A upload");
    ctx->st_h2d += (size_t)m * K * 4;
    tmark("A up", d->h2d);
    CAFXG_TRY(stream_after_pooled(d, cs, d->h2d));
    if (i >= 2)
      cudaStreamWaitEvent(cs, ev_down[i - 2], 0);  // C slot drained
    e = raw ? sgemm_tc_lo(dA[slot], (int)K, (int)m, (int)K, Al, d->sms, cs)
            : sgemm_tc_split_a(dA[slot], (int)K, (int)m, (int)K, Ah, Al, cs);
    cudaEventRecord(mk(ev_split), cs);
    if (e == 0) {
      int sp = g.splits ? (int)g.splits : sgemm_tc_splits((int)m, (int)N, (int)K, d->sms, bn);
      if (raw && sp > splits_max)
        sp = splits_max;  // (the workspace is sized for R-row blocks)
      e = sgemm_tc_gemm_maps(raw ? &rmaps[slot] : &maps, dC[slot], (int)m, (int)N, (int)K,
                             (int)N, cs, sp, 0, 0, raw ? wsk : nullptr);
    }
    if (e != 0)
      status = cuda_status((cudaError_t)e, "sgemm: 3xtf32 launch");
    ctx->st_launches += 2;
    mark_used(ctx, d);
    tmark("gemm", cs);
    cudaEventRecord(mk(ev_gemm), cs);
    cudaStreamWaitEvent(d->d2h, ev_gemm.back(), 0);
    if (status == CAFXG_OK)
      status = cuda_status(
          g.ldc == N ? cudaMemcpyAsync(C + (size_t)(r0 + b0) * g.ldc, dC[slot], (size_t)m * N * 4,
                                       cudaMemcpyDeviceToHost, d->d2h)
                     : cudaMemcpy2DAsync(C + (size_t)(r0 + b0) * g.ldc, (size_t)g.ldc * 4,
                                         dC[slot], N * 4, N * 4, m, cudaMemcpyDeviceToHost,
                                         d->d2h),
          "sgemm: C download");
    ctx->st_d2h += (size_t)m * N * 4;
    tmark("C down", d->d2h);
    cudaEventRecord(mk(ev_down), d->d2h);
  }
  if (!tev.empty()) {
    const double t_host1 = trace_now_ms();
    cudaEventSynchronize(tev.back().second);
    const double t_seen = trace_now_ms();
    fprintf(stderr, "cafxg sgemm trace: host enqueue %.3f ms, sync seen at %.3f ms; device:",
            t_host1 - t_host0, t_seen - t_host0);
    for (auto& [what, e] : tev) {
      float t = 0;
      cudaEventElapsedTime(&t, tev[0].second, e);
      fprintf(stderr, " %s %.3f", what, t);
    }
    fprintf(stderr, "\n");
    for (auto& pe : tev)
      cudaEventDestroy(pe.second);
  }
  // everything is released on the download stream, which by now follows
  // every upload and kernel of this request
  CAFXG_TRY(stream_after_pooled(d, d->d2h, cs));
  // every wait on these records is enqueued: back to the pool
  for (auto* v : {&ev_split, &ev_gemm, &ev_down})
    for (auto ev : *v)
      if (ev)
        d->ev_pool.push_back(ev);
  return status;
}

// Large single-device host requests: a 2D wavefront over C blocks. A's row
// blocks and B's column blocks go up interleaved (A0, B0, A1, B1, ...); each
// block is split (tf32 hi/lo; B^T) as it lands, and every C block (i, j)
// whose A_i and B_j are both resident is multiplied at once and downloaded
// on the copy stream. The row-block pipeline needs all of B before its first
// GEMM (1 GiB, ~20 ms over PCIe at 16384^3); here compute follows the
// uploads one block behind, so the request approaches the 2 GiB upload time.
bool sgemm_tiled2d_eligible(const cafxg_sgemm_desc& g) {
  static const bool on = [] {
    const char* e = getenv("CAFXG_SGEMM_2D");
    return !(e && e[0] == '0');
  }();
  static const uint32_t min_dim = [] {  // CAFXG_SGEMM_2D_MIN: experiments only
    const char* e = getenv("CAFXG_SGEMM_2D_MIN");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? (uint32_t)v : 8192u;
  }();
  return on && g.mode != CAFXG_SGEMM_FFMA && g.M >= min_dim && g.N >= min_dim &&
         g.M % 128 == 0 &&
         g.N % 256 == 0 && sgemm_tc_supported(128, 256, g.K, g.K, g.N, g.N);
}

int sgemm_tiled2d_device(cafxg_ctx* ctx, Device* d, const cafxg_sgemm_desc& g,
                                const float* A, const float* B, float* C) {
  const size_t M = g.M, N = g.N, K = g.K;
  static const uint32_t div = [] {  // blocks per dimension (CAFXG_SGEMM_2D_DIV)
    const char* e = getenv("CAFXG_SGEMM_2D_DIV");
    const int v = e ? atoi(e) : 0;
    return v >= 2 && v <= 64 ? (uint32_t)v : 8u;
  }();
  const uint32_t Mb = (uint32_t)((M / div + 127) / 128 * 128);
  // column blocks sized so a block's C tiles (128 x 256 each, one CTA per
  // tile) come close to one full wave of SMs: 2048 x 2304 blocks are 144
  // tiles on 148 SMs where 2048 x 2048 were 128
  uint32_t Nb = (uint32_t)((N / div + 255) / 256 * 256);
  {
    const uint32_t rows_t = Mb / 128;
    uint32_t cols_t = std::max<uint32_t>(1, (uint32_t)d->sms / std::max<uint32_t>(1, rows_t));
    if (cols_t * 256 >= Nb && cols_t * 256 < 2 * Nb)
      Nb = std::min<uint32_t>(cols_t * 256, (uint32_t)N);
  }
  const uint32_t nbm = (uint32_t)((M + Mb - 1) / Mb), nbn = (uint32_t)((N + Nb - 1) / Nb);
  cudaStream_t cs = d->compute;
  float *dA = nullptr, *dB = nullptr, *Ah = nullptr, *Al = nullptr, *Bh = nullptr,
        *Bl = nullptr, *dC = nullptr;
  CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dA, M * K * 4, cs));
  CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dB, K * N * 4, cs));
  CAFXG_CUDA_TRY(cudaMallocAsync((void**)&Ah, M * K * 4, cs));
  CAFXG_CUDA_TRY(cudaMallocAsync((void**)&Al, M * K * 4, cs));
  CAFXG_CUDA_TRY(cudaMallocAsync((void**)&Bh, N * K * 4, cs));
  CAFXG_CUDA_TRY(cudaMallocAsync((void**)&Bl, N * K * 4, cs));
  CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dC, M * N * 4, cs));
  SgemmTcMaps maps;  // whole Ah/Al and Bh/Bl; blocks address rows by offset
  if (int me = sgemm_tc_make_maps(Ah, Al, (int)M, Bh, Bl, (int)N, (int)K, 256, &maps))
    return cuda_status((cudaError_t)me, "sgemm: tensor maps");
  // the same operands for the CTA-pair kernel (blocks of whole 256 x 256
  // pair tiles whose grid needs no split-K)
  SgemmTcMaps pmaps;
  const bool pair_ok =
      sgemm_tc_make_pair_maps(Ah, Al, (int)M, Bh, Bl, (int)N, (int)K, &pmaps) == 0;
  CAFXG_TRY(stream_after_pooled(d, d->h2d, cs));  // buffers exist before uploads
  // CAFXG_TRACE=1: completion times of uploads, GEMM blocks and downloads
  std::vector<std::pair<char, cudaEvent_t>> tev;
  auto tmark = [&](char what, cudaStream_t sm) {
    if (!trace_on())
      return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, sm);
    tev.emplace_back(what, e);
  };
  tmark('S', d->h2d);
  std::vector<cudaEvent_t> evs;
  auto ev_on = [&](cudaStream_t sm) {
    cudaEvent_t e = pooled_event(d);
    cudaEventRecord(e, sm);
    evs.push_back(e);
    return e;
  };
  int status = CAFXG_OK;
  uint32_t na = 0, nb = 0;  // A row blocks / B column blocks resident
  auto gemm_block = [&](uint32_t i, uint32_t j) {
    const uint32_t m0 = i * Mb, n0 = j * Nb;
    const uint32_t mi = (uint32_t)std::min<size_t>(Mb, M - m0);
    const uint32_t nj = (uint32_t)std::min<size_t>(Nb, N - n0);
    float* cblk = dC + (size_t)m0 * N + n0;
    const bool pair = pair_ok && !g.splits && mi % 256 == 0 && nj % 256 == 0 &&
                      sgemm_tc_pair_wanted((int)mi, (int)nj, (int)K, d->sms);
    int e = sgemm_tc_gemm_maps(pair ? &pmaps : &maps, cblk, (int)mi, (int)nj, (int)K, (int)N,
                               cs,
                               pair ? 1
                               : g.splits
                                   ? (int)g.splits
                                   : sgemm_tc_splits((int)mi, (int)nj, (int)K, d->sms, 256),
                               (int)m0, (int)n0);
    ctx->st_launches++;
    mark_used(ctx, d);
    tmark('G', cs);
    if (e != 0)
      return cuda_status((cudaError_t)e, "sgemm: 3xtf32 block launch");
    cudaStreamWaitEvent(d->d2h, ev_on(cs), 0);
    ctx->st_d2h += (size_t)mi * nj * 4;
    const int st = cuda_status(cudaMemcpy2DAsync(C + (size_t)m0 * g.ldc + n0, (size_t)g.ldc * 4,
                                                 cblk, N * 4, (size_t)nj * 4, mi,
                                                 cudaMemcpyDeviceToHost, d->d2h),
                               "sgemm: C block download");
    tmark('D', d->d2h);
    return st;
  };
  for (uint32_t t = 0; t < std::max(nbm, nbn) && status == CAFXG_OK; ++t) {
    if (t < nbm) {  // A row block t
      const uint32_t m0 = t * Mb, mi = (uint32_t)std::min<size_t>(Mb, M - m0);
      status = cuda_status(cudaMemcpy2DAsync(dA + (size_t)m0 * K, K * 4, A + (size_t)m0 * g.lda,
                                             (size_t)g.lda * 4, K * 4, mi,
                                             cudaMemcpyHostToDevice, d->h2d),
                           "sgemm: A block upload");
      ctx->st_h2d += (size_t)mi * K * 4;
      tmark('A', d->h2d);
      if (status != CAFXG_OK)
        break;
      cudaStreamWaitEvent(cs, ev_on(d->h2d), 0);
      int e = sgemm_tc_split_a(dA + (size_t)m0 * K, (int)K, (int)mi, (int)K, Ah + (size_t)m0 * K,
                               Al + (size_t)m0 * K, cs);
      ctx->st_launches++;
      if (e != 0) {
        status = cuda_status((cudaError_t)e, "sgemm: A split");
        break;
      }
      ++na;
      for (uint32_t j = 0; j < nb && status == CAFXG_OK; ++j)
        status = gemm_block(t, j);
    }
    if (t < nbn && status == CAFXG_OK) {  // B column block t
      const uint32_t n0 = t * Nb, nj = (uint32_t)std::min<size_t>(Nb, N - n0);
      status = cuda_status(cudaMemcpy2DAsync(dB + n0, N * 4, B + n0, (size_t)g.ldb * 4,
                                             (size_t)nj * 4, K, cudaMemcpyHostToDevice, d->h2d),
                           "sgemm: B block upload");
      ctx->st_h2d += K * nj * 4;
      tmark('B', d->h2d);
      if (status != CAFXG_OK)
        break;
      cudaStreamWaitEvent(cs, ev_on(d->h2d), 0);
      int e = sgemm_tc_split_b(dB + n0, (int)N, (int)K, (int)nj, Bh + (size_t)n0 * K,
                               Bl + (size_t)n0 * K, cs);
      ctx->st_launches++;
      if (e != 0) {
        status = cuda_status((cudaError_t)e, "sgemm: B split");
        break;
      }
      ++nb;
      for (uint32_t i = 0; i < na && status == CAFXG_OK; ++i)
        status = gemm_block(i, t);
    }
  }
  if (!tev.empty()) {
    cudaEventSynchronize(tev.back().second);
    fprintf(stderr, "cafxg sgemm 2d trace (ms):");
    for (auto& [w, e] : tev) {
      float t = 0;
      cudaEventElapsedTime(&t, tev[0].second, e);
      fprintf(stderr, " %c%.2f", w, t);
    }
    fprintf(stderr, "\n");
    for (auto& pe : tev)
      cudaEventDestroy(pe.second);
  }
  CAFXG_TRY(stream_after_pooled(d, d->d2h, cs));
  for (float* p : {dA, dB, Ah, Al, Bh, Bl, dC})
    cudaFreeAsync(p, d->d2h);
  for (auto e : evs)
    if (e)
      d->ev_pool.push_back(e);
  return status;
}

// Host-to-host sgemm. One device: H2D A,B -> GEMM -> D2H C. G devices: A is
// split into row blocks; each device uploads 1/G of B's rows and an NCCL
// all-gather over NVLink completes B everywhere; each device returns its C
// rows.
int sgemm_submit_impl(cafxg_ctx* ctx, const cafxg_sgemm_desc* desc,
                             const float* A, const float* B, float* C,
                             cafxg_done_fn done, void* user) {
  NvtxRange nvtx_range("cafxg.sgemm.submit");
  if (!ctx || !desc)
    return fail(CAFXG_E_CONFIG, "sgemm_submit: null argument");
  cafxg_sgemm_desc g = *desc;
  CAFXG_TRY(validate_sgemm(g));
  CAFXG_TRY(check_alive(ctx));
  if ((g.M && g.K && !A) || (g.K && g.N && !B) || (g.M && g.N && !C))
    return fail(CAFXG_E_CONFIG, "sgemm_submit: null matrix");
  size_t G = ctx->devs.size();
  // devices used: only split when every block gets rows and K divides evenly
  size_t use = 1;
  bool nccl = false;
  if (G > 1 && g.M >= G * 128 && g.K % G == 0 && g.ldb == g.N) {
    use = G;
    // the GEMM that reads B's slices from the peers in place (above)
    const uint32_t rp = (uint32_t)((g.M + use - 1) / use);
    const uint32_t rows_per = (rp + 127) / 128 * 128;
    if (p2p_eligible(ctx, g, rows_per)) {
      clear_last_error();
      Join* join = new Join;
      join->done = done;
      join->user = user;
      join->remaining = (int)use;
      ctx->st_requests++;
      ctx->st_p2p++;
      return sgemm_p2p_submit(ctx, g, A, B, C, rows_per, join);
    }
    clear_last_error();
    // NCCL all-gather over NVLink; without it (virtual devices, or NCCL not
    // loadable) the slices are replicated by peer copies on the copy engines
    nccl = ensure_nccl(ctx) == CAFXG_OK;
    clear_last_error();
  } else if (G == 1 && nccl_selftest()) {
    // CAFXG_NCCL_SELFTEST=1: a one-device context runs B through the same
    // NCCL calls (a one-rank communicator, in-place all-gather), so the NCCL
    // branch is exercised on a one-GPU box; failing to set it up is an error
    CAFXG_TRY(ensure_nccl(ctx));
    nccl = true;
  }
  Join* join = new Join;
  join->done = done;
  join->user = user;
  join->remaining = (int)use;
  ctx->st_requests++;
  if (use == 1 && !nccl && sgemm_tiled2d_eligible(g)) {
    Device* d = ctx->devs[0].get();
    std::lock_guard<std::mutex> lk(d->submit_mu);
    cudaSetDevice(d->ordinal);
    int s = sgemm_tiled2d_device(ctx, d, g, A, B, C);
    // a failure is reported after the queued work: it may still read the
    // host buffers
    if (s != CAFXG_OK)
      push_completion(ctx, d, d->d2h, [join, s](int) { join->part_done(s); });
    else
      push_completion(ctx, d, d->d2h, [join](int st) { join->part_done(st); });
    return CAFXG_OK;
  }
  const size_t bytesB = (size_t)g.K * g.ldb * 4;
  const uint32_t rows_per = (uint32_t)((g.M + use - 1) / use);
  // allocation + upload of B slices on every used device
  std::vector<float*> dB(use, nullptr);
  std::vector<std::unique_lock<std::mutex>> locks;
  for (size_t k = 0; k < use; ++k)
    locks.emplace_back(ctx->devs[k]->submit_mu);
  int status = CAFXG_OK;
  const bool defer_b =
      use == 1 && !nccl && g.M && g.ldb == g.N && sgemm_pipeline_eligible(g, g.M);
  for (size_t k = 0; k < use && status == CAFXG_OK; ++k) {
    Device* d = ctx->devs[k].get();
    cudaSetDevice(d->ordinal);
    if (cudaMallocAsync((void**)&dB[k], std::max<size_t>(bytesB, 4), d->compute) != cudaSuccess) {
      status = cuda_status(cudaGetLastError(), "sgemm: device B allocation");
      break;
    }
    if (defer_b)
      continue;  // uploaded by sgemm_pipeline_device on the upload stream
    size_t k0 = use == 1 ? 0 : (size_t)g.K / use * k;
    size_t kn = use == 1 ? g.K : (size_t)g.K / use;
    if (kn && cudaMemcpyAsync(dB[k] + k0 * g.ldb, B + k0 * g.ldb, kn * g.ldb * 4,
                              cudaMemcpyHostToDevice, d->compute) != cudaSuccess)
      status = cuda_status(cudaGetLastError(), "sgemm: B upload");
    ctx->st_h2d += kn * g.ldb * 4;
  }
  if (status == CAFXG_OK && use > 1 && !nccl) {
    // each device pulls the other devices' slices once they are uploaded
    std::vector<cudaEvent_t> up(use, nullptr);
    for (size_t k = 0; k < use && status == CAFXG_OK; ++k) {
      cudaSetDevice(ctx->devs[k]->ordinal);
      if (cudaEventCreateWithFlags(&up[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventRecord(up[k], ctx->devs[k]->compute) != cudaSuccess)
        status = cuda_status(cudaGetLastError(), "sgemm: B slice event");
    }
    const size_t cnt = (size_t)g.K / use * g.ldb;
    for (size_t k = 0; k < use && status == CAFXG_OK; ++k) {
      Device* d = ctx->devs[k].get();
      cudaSetDevice(d->ordinal);
      for (size_t j = 0; j < use && status == CAFXG_OK; ++j) {
        if (j == k)
          continue;
        cudaStreamWaitEvent(d->compute, up[j], 0);
        status = cuda_status(cudaMemcpyPeerAsync(dB[k] + cnt * j, d->ordinal, dB[j] + cnt * j,
                                                 ctx->devs[j]->ordinal, cnt * 4, d->compute),
                             "sgemm: B slice peer copy");
      }
    }
    // a device's own slice buffer must outlive the peers' reads of it
    std::vector<cudaEvent_t> pulled(use, nullptr);
    for (size_t k = 0; k < use && status == CAFXG_OK; ++k) {
      cudaSetDevice(ctx->devs[k]->ordinal);
      cudaEventCreateWithFlags(&pulled[k], cudaEventDisableTiming);
      cudaEventRecord(pulled[k], ctx->devs[k]->compute);
    }
    for (size_t k = 0; k < use && status == CAFXG_OK; ++k) {
      cudaSetDevice(ctx->devs[k]->ordinal);
      for (size_t j = 0; j < use; ++j)
        if (j != k)
          cudaStreamWaitEvent(ctx->devs[k]->compute, pulled[j], 0);
    }
    for (auto* v : {&up, &pulled})
      for (auto ev : *v)
        if (ev)
          cudaEventDestroy(ev);
  }
  if (status == CAFXG_OK && nccl) {
    ctx->nccl.GroupStart();
    for (size_t k = 0; k < use; ++k) {
      size_t cnt = (size_t)g.K / use * g.ldb;
      ctx->nccl.AllGather(dB[k] + cnt * k, dB[k], cnt, ncclFloat32, ctx->comms[k],
                          ctx->devs[k]->compute);
    }
    if (ctx->nccl.GroupEnd() != ncclSuccess)
      status = fail(CAFXG_E_DOWN, "sgemm: NCCL all-gather of B failed");
    else
      ctx->st_nccl += use;
  }
  for (size_t k = 0; k < use; ++k) {
    Device* d = ctx->devs[k].get();
    cudaSetDevice(d->ordinal);
    int s = status;
    uint32_t r0 = (uint32_t)std::min<uint64_t>(g.M, (uint64_t)rows_per * k);
    uint32_t r1 = (uint32_t)std::min<uint64_t>(g.M, (uint64_t)rows_per * (k + 1));
    cafxg_sgemm_desc part = g;
    part.M = r1 - r0;
    part.lda = g.K;
    part.ldc = g.N;
    float *dA = nullptr, *dC = nullptr;
    if (s == CAFXG_OK && part.M && g.ldb == g.N && sgemm_pipeline_eligible(g, part.M)) {
      s = sgemm_pipeline_device(ctx, d, g, A, dB[k], C, r0, r1, defer_b ? B : nullptr);
      cudaFreeAsync(dB[k], d->d2h);
      if (s != CAFXG_OK)
        push_completion(ctx, d, d->d2h, [join, s](int) { join->part_done(s); });
      else
        push_completion(ctx, d, d->d2h, [join](int st) { join->part_done(st); });
      continue;
    }
    if (s == CAFXG_OK && part.M) {
      if (cudaMallocAsync((void**)&dA, (size_t)part.M * g.K * 4 + 4, d->compute) != cudaSuccess ||
          cudaMallocAsync((void**)&dC, (size_t)part.M * g.N * 4 + 4, d->compute) != cudaSuccess)
        s = cuda_status(cudaGetLastError(), "sgemm: device allocation");
      if (s == CAFXG_OK && g.K) {
        if (g.lda == g.K)
          s = cuda_status(cudaMemcpyAsync(dA, A + (size_t)r0 * g.lda, (size_t)part.M * g.K * 4,
                                          cudaMemcpyHostToDevice, d->compute), "sgemm: A upload");
        else
          s = cuda_status(cudaMemcpy2DAsync(dA, (size_t)g.K * 4, A + (size_t)r0 * g.lda,
                                            (size_t)g.lda * 4, (size_t)g.K * 4, part.M,
                                            cudaMemcpyHostToDevice, d->compute), "sgemm: A upload");
        ctx->st_h2d += (size_t)part.M * g.K * 4;
      }
      if (s == CAFXG_OK)
        s = sgemm_on_device(ctx, d, part, dA, dB[k], dC, d->compute);
      if (s == CAFXG_OK) {
        s = cuda_status(cudaMemcpy2DAsync(C + (size_t)r0 * g.ldc, (size_t)g.ldc * 4, dC,
                                          (size_t)g.N * 4, (size_t)g.N * 4, part.M,
                                          cudaMemcpyDeviceToHost, d->compute), "sgemm: C download");
        ctx->st_d2h += (size_t)part.M * g.N * 4;
      }
    }
    if (dA) cudaFreeAsync(dA, d->compute);
    if (dC) cudaFreeAsync(dC, d->compute);
    if (dB[k]) cudaFreeAsync(dB[k], d->compute);
    // a failure is still routed through the completion thread
    if (s != CAFXG_OK)
      push_completion(ctx, d, d->compute, [join, s](int) { join->part_done(s); });
    else
      push_completion(ctx, d, d->compute, [join](int st) { join->part_done(st); });
  }
  return CAFXG_OK;
}

}  // namespace cafxg

using namespace cafxg;

extern "C" {

int cafxg_sgemm_submit(cafxg_ctx* ctx, const cafxg_sgemm_desc* d, const float* A,
                       const float* B, float* C, cafxg_done_fn done, void* user) {
  try {
    return sgemm_submit_impl(ctx, d, A, B, C, done, user);
  } catch (const std::exception& ex) {
    return fail(CAFXG_E_CONFIG, "sgemm_submit: %s", ex.what());
  }
}

int cafxg_sgemm(cafxg_ctx* ctx, const cafxg_sgemm_desc* d, const float* A, const float* B,
                float* C) try {
  Waiter w;
  int s = cafxg_sgemm_submit(ctx, d, A, B, C, &Waiter::cb, &w);
  if (s != CAFXG_OK)
    return s;
  return w.wait();
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_sgemm: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_sgemm: unknown exception");
}

int cafxg_sgemm_device(cafxg_ctx* ctx, int device, const cafxg_sgemm_desc* desc,
                       const float* A, const float* B, float* C, void* stream) try {
  if (!ctx || !desc || device < 0 || device >= (int)ctx->devs.size())
    return fail(CAFXG_E_CONFIG, "sgemm_device: bad argument");
  cafxg_sgemm_desc g = *desc;
  CAFXG_TRY(validate_sgemm(g));
  CAFXG_TRY(check_alive(ctx));
  Device* d = ctx->devs[device].get();
  cudaSetDevice(d->ordinal);
  return sgemm_on_device(ctx, d, g, A, B, C, stream ? (cudaStream_t)stream : d->compute);
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_sgemm_device: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_sgemm_device: unknown exception");
}

}  // extern "C"
