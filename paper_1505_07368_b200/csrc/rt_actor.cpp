// libcafxg.so host runtime, compute actors: spawn_cl-style actors
// (cafxg_spawn / cafxg_actor_enqueue), the MPSC inbox, the batching
// dispatcher, batch launches with direct or scattered replies, and the reply
// callback threads.
#include "runtime_internal.hpp"

namespace cafxg {

// ---- compute actors + dispatcher ---------------------------------------------------

enum class Kernel : uint32_t { mandelbrot = 1, matrix_multiply = 2 };

}  // namespace cafxg

struct cafxg_actor {
  cafxg_ctx* ctx;
  Kernel kernel;
  uint64_t dims[3] = {0, 0, 0};
  size_t ndims = 0;
  std::atomic<bool> alive{true};
  std::atomic<int> refs{1};
  std::atomic<uint64_t> pending{0};
  cafxg_tuning tune{};  // spawn_cl tuning overload (zeros: backend defaults)
};

namespace cafxg {
// replies delivered together with the current done callback on this thread
// (cafxg_completion_batch); 1 outside finish_batch's slices
thread_local size_t t_completion_batch = 1;

// requests of actors spawned with different tuning never share a launch
static bool same_tuning(const cafxg_actor* a, const cafxg_actor* b) {
  return a == b || std::memcmp(&a->tune, &b->tune, sizeof(cafxg_tuning)) == 0;
}
}  // namespace cafxg

struct Request {
  const cafxg_mandel_desc& tile(size_t i) const { return i == 0 ? tile0 : more[i - 1]; }
  Request* next = nullptr;
  cafxg_actor* actor = nullptr;
  // mandelbrot tiles: the first inline (a storm request is one tile, so the
  // dispatcher touches one cache-resident node per request), the rest behind
  cafxg_mandel_desc tile0{};
  std::vector<cafxg_mandel_desc> more;
  uint32_t ntiles = 0;
  int precision = 0;
  const float* a = nullptr;              // matrix_multiply
  const float* b = nullptr;
  void* out = nullptr;
  size_t out_bytes = 0;
  uint64_t pixels = 0;
  uint32_t max_iter = 0;
  bool exact = false;       // needs the 8-op escape step (tiny |ci| rows)
  bool out_pinned = false;  // reply buffer is device-mapped pinned memory
  cafxg_done_fn done = nullptr;
  void* user = nullptr;
};

namespace cafxg {

void actor_unref(cafxg_actor* a) {
  if (a->refs.fetch_sub(1) == 1)
    delete a;
}

// Completes one actor request: the caller's callback, then the bookkeeping.
// `account` = false when the caller settles the context counters for a whole
// batch at once (st_requests / actor_open / the sync notification).
void finish_request(Request* r, int status, bool account = true) {
  cafxg_actor* a = r->actor;
  cafxg_ctx* ctx = a->ctx;
  if (r->done)
    r->done(r->user, status);
  a->pending.fetch_sub(1);
  actor_unref(a);
  delete r;
  if (account) {
    ctx->st_requests++;
    ctx->actor_open.fetch_sub(1);
    ctx->sync_cv.notify_all();
  }
}

// Runs a finished batch's reply callbacks. Large batches are split across the
// context's callback threads (the per-request callback -- a cafx `deliver`
// in the adapter -- would otherwise serialise on one completion thread).
void finish_batch(cafxg_ctx* ctx, std::vector<Request*> batch, uint32_t* bounce,
                         int status);

// Callback thread: runs reply jobs (slices of large batches, copy pieces).
void callback_loop(cafxg_ctx* ctx) {
  while (true) {
    std::function<void()> job;
    {
      std::unique_lock<std::mutex> lk(ctx->cb_mu);
      ctx->cb_cv.wait(lk, [&] { return ctx->cb_stop || !ctx->cb_q.empty(); });
      if (ctx->cb_q.empty())
        return;
      job = std::move(ctx->cb_q.front());
      ctx->cb_q.pop_front();
    }
    run_guarded("reply callback", job);
  }
}

void finish_batch(cafxg_ctx* ctx, std::vector<Request*> batch, uint32_t* bounce,
                         int status) {
  constexpr size_t kSlice = 1024;
  const size_t n = batch.size();
  // src: the staging buffer to copy replies out of (nullptr: already placed)
  auto run_slice = [ctx, status](Request* const* rs, size_t cnt, uint64_t pix_off,
                                 const uint32_t* src) {
    uint64_t o = pix_off;
    t_completion_batch = cnt;  // cafxg_completion_batch() inside the callbacks
    for (size_t i = 0; i < cnt; ++i) {
      Request* r = rs[i];
      if (src && status == CAFXG_OK)
        std::memcpy(r->out, src + o, r->pixels * 4);
      o += r->pixels;
      finish_request(r, status, false);
    }
    t_completion_batch = 1;
    ctx->st_requests += cnt;
    ctx->actor_open.fetch_sub(cnt);
    ctx->sync_cv.notify_all();
  };
  uint64_t total_px = 0;
  for (Request* r : batch)
    total_px += r->pixels;
  constexpr uint64_t kPiece = 1 << 20;  // bytes per copy piece
  if (bounce && status == CAFXG_OK && n <= kSlice && total_px * 4 >= 4 * kPiece &&
      !ctx->cb_threads.empty()) {
    // few large pageable replies (e.g. one 1920x1080 image): the staging
    // copy-out is split into 1 MiB pieces over the callback threads and this
    // thread; the last piece to finish completes the requests
    struct Piece {
      void* dst;
      const void* src;
      size_t bytes;
    };
    auto pieces = std::make_shared<std::vector<Piece>>();
    uint64_t o = 0;
    for (Request* r : batch) {
      const size_t bytes = r->pixels * 4;
      for (size_t b = 0; b < bytes; b += kPiece)
        pieces->push_back({(char*)r->out + b, (const char*)(bounce + o) + b,
                           std::min<size_t>(kPiece, bytes - b)});
      o += r->pixels;
    }
    auto shared = std::make_shared<std::vector<Request*>>(std::move(batch));
    auto left = std::make_shared<std::atomic<size_t>>(pieces->size());
    auto piece_job = [ctx, shared, pieces, left, bounce, run_slice](size_t i) {
      const Piece& p = (*pieces)[i];
      std::memcpy(p.dst, p.src, p.bytes);
      if (left->fetch_sub(1) == 1) {
        run_slice(shared->data(), shared->size(), 0, nullptr);
        ctx->pinned.free(bounce);
      }
    };
    {
      std::lock_guard<std::mutex> g(ctx->cb_mu);
      for (size_t i = 1; i < pieces->size(); ++i)
        ctx->cb_q.push_back([piece_job, i] { piece_job(i); });
    }
    ctx->cb_cv.notify_all();
    piece_job(0);
    return;
  }
  if (n <= kSlice || ctx->cb_threads.empty()) {
    run_slice(batch.data(), n, 0, bounce);
    if (bounce)
      ctx->pinned.free(bounce);
    return;
  }
  // slices run on the callback threads; the last one frees the bounce buffer
  auto shared = std::make_shared<std::vector<Request*>>(std::move(batch));
  auto left = std::make_shared<std::atomic<size_t>>((n + kSlice - 1) / kSlice);
  uint64_t pix = 0;
  std::vector<std::function<void()>> jobs;
  for (size_t b = 0; b < n; b += kSlice) {
    size_t cnt = std::min(kSlice, n - b);
    jobs.push_back([ctx, shared, left, b, cnt, pix, bounce, run_slice] {
      run_slice(shared->data() + b, cnt, pix, bounce);
      if (left->fetch_sub(1) == 1 && bounce)
        ctx->pinned.free(bounce);
    });
    for (size_t i = b; i < b + cnt; ++i)
      pix += (*shared)[i]->pixels;
  }
  {
    std::lock_guard<std::mutex> g(ctx->cb_mu);
    for (auto& j : jobs)
      ctx->cb_q.push_back(std::move(j));
  }
  ctx->cb_cv.notify_all();
}

inline uint64_t now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// One batch of Mandelbrot requests (same precision) on one device: one launch
// over every tile of every request into a device staging slot; small batches
// into pinned replies are then copied out by that kernel itself (direct
// reply), others by one scatter launch straight into the pinned reply buffers
// (or one D2H into a pinned bounce buffer + host memcpy for pageable replies).
void run_mandel_batch(cafxg_ctx* ctx, Device* d, std::vector<Request*> batch) {
  NvtxRange nvtx_range("cafxg.actor.batch");
  const double t_begin = trace_now_ms();
  uint64_t ph = now_ns();
  auto phase = [&](int i) {
    const uint64_t t = now_ns();
    ctx->st_phase_ns[i] += t - ph;
    ph = t;
  };
  cudaSetDevice(d->ordinal);
  std::lock_guard<std::mutex> g(d->submit_mu);
  const double t_lock = trace_now_ms();
  uint64_t px = 0;
  uint32_t maxit = 0;
  bool exact = false;
  int prec = batch[0]->precision;
  bool all_pinned = true;
  size_t ntiles = 0;
  for (Request* r : batch) {
    px += r->pixels;
    maxit = std::max(maxit, r->max_iter);
    exact = exact || r->exact;
    ntiles += r->ntiles;
    all_pinned = all_pinned && r->out_pinned;
  }
  int status = CAFXG_OK;
  uint32_t* dout = nullptr;
  uint32_t* bounce = nullptr;
  CopySeg* dsegs = nullptr;
  auto fail_all = [&](int s) {
    std::string err = t_last_error;
    for (Request* r : batch)
      push_completion(ctx, d, d->compute, [r, s](int) { finish_request(r, s); });
    t_last_error = err;
  };
  const uint32_t slot = d->stage_next++ % kMaxInflight;
  // consecutive batches alternate between the two compute streams: a small
  // batch's kernel is latency-bound (fp64 storm tiles: ~16 us for 256
  // dependent iterations on a fraction of the SMs), so batches in flight
  // overlap instead of queueing behind each other
  cudaStream_t ks = (slot & 1) ? d->compute2 : d->compute;
  // Direct reply (mandel_kernel / mandel_deferred_kernel copy each finished
  // tile to its pinned reply themselves): small batches whose replies are all
  // device-mapped pinned memory. Saves the reply-scatter launch and the
  // copy-stream ordering on the dispatcher, and the launch gap on the device.
  bool direct = all_pinned && direct_reply_enabled() && ntiles <= (size_t)kInlineTiles &&
                px < (1ull << kDirectShift);
  for (Request* r : batch) {
    direct = direct && r->max_iter == maxit && (reinterpret_cast<uintptr_t>(r->out) & 15) == 0;
    for (uint32_t k = 0; direct && k < r->ntiles; ++k) {
      const cafxg_mandel_desc& t = r->tile(k);
      const uint64_t tp = (uint64_t)t.nrows * t.ncols;
      // one launch (one max_iter group) covers a direct batch: a request
      // whose tiles differ in max_iter takes the scatter path
      direct = tp % 4 == 0 && tp <= kDirectTilePx && t.max_iter == maxit;
    }
  }
  if (!d->stage[0]) {
    // first batch on this device: the whole ring at the batch cap, so later
    // batches never allocate (one request above the cap still grows its slot)
    for (int i = 0; i < kMaxInflight; ++i) {
      const size_t cap = kMaxBatchPx * 4 + kStageTail;
      if (cudaMalloc((void**)&d->stage[i], cap) == cudaSuccess &&
          cudaMemset(d->stage[i] + cap - kStageTail, 0, kStageTail) == cudaSuccess &&
          // the legacy stream's memset is not ordered before the non-blocking
          // compute streams: wait for it
          cudaStreamSynchronize(0) == cudaSuccess) {
        d->stage_cap[i] = cap;
      } else {
        cudaGetLastError();
        d->stage[i] = nullptr;
        break;
      }
    }
  }
  {
    const size_t need = px * 4 + kStageTail;
    if (d->stage_cap[slot] < need) {
      // growth (warm-up): the old buffer may still feed an earlier batch
      if (d->stage[slot]) {
        cudaStreamSynchronize(d->compute);
        cudaStreamSynchronize(d->compute2);
        cudaStreamSynchronize(d->d2h);
        cudaFree(d->stage[slot]);
        d->stage[slot] = nullptr;
        d->stage_cap[slot] = 0;
      }
      size_t cap = std::max<size_t>(need, kMaxBatchPx * 4 + kStageTail);
      if (cudaMalloc((void**)&d->stage[slot], cap) != cudaSuccess ||
          cudaMemset(d->stage[slot] + cap - kStageTail, 0, kStageTail) != cudaSuccess ||
          cudaStreamSynchronize(0) != cudaSuccess) {
        d->stage[slot] = nullptr;
        fail_all(cuda_status(cudaGetLastError(), "batch staging allocation"));
        return;
      }
      d->stage_cap[slot] = cap;
    }
    if (!d->stage_ev[slot] &&
        cudaEventCreateWithFlags(&d->stage_ev[slot], cudaEventDisableTiming) != cudaSuccess) {
      d->stage_ev[slot] = nullptr;
      fail_all(cuda_status(cudaGetLastError(), "batch staging event"));
      return;
    }
    // the copy-out of the batch that used this slot before must be done
    // reading it (recorded on the copy stream). A slot always runs on the
    // same compute stream (kMaxInflight is even), so after a direct-reply
    // batch the order is implied.
    if (d->stage_on_copy[slot])
      cudaStreamWaitEvent(ks, d->stage_ev[slot], 0);
    d->stage_on_copy[slot] = !direct;
    dout = reinterpret_cast<uint32_t*>(d->stage[slot]);
  }
  std::vector<MTile> mt;
  mt.reserve(ntiles);
  std::vector<CopySeg> segs;
  uint32_t chunks = 0;
  uint64_t off = 0;
  for (Request* r : batch) {
    uint64_t roff = off;
    for (uint32_t k = 0; k < r->ntiles; ++k) {
      const cafxg_mandel_desc& t = r->tile(k);
      MTile m;
      fill_mtile(m, t, off, chunks);
      if (direct)
        m.reply = static_cast<uint32_t*>(r->out) + (off - roff);
      mt.push_back(m);
      uint64_t tp = (uint64_t)t.nrows * t.ncols;
      chunks += tile_chunks(t.nrows, t.ncols, t.precision);
      off += tp;
    }
    segs.push_back(CopySeg{dout + roff, r->out, (off - roff) * 4});
  }
  const double t_built = trace_now_ms();
  phase(0);
  // CAFXG_TRACE: device-side timestamps of this batch (kernel start/end,
  // copy-out end), reported against a per-device reference event
  cudaEvent_t tev[3] = {};
  if (trace_on()) {
    if (!d->trace_ref) {
      cudaEventCreate(&d->trace_ref);
      cudaEventRecord(d->trace_ref, ks);
      cudaEventSynchronize(d->trace_ref);
      d->trace_ref_ms = trace_now_ms();
    }
    for (auto& e : tev)
      cudaEventCreate(&e);
    cudaEventRecord(tev[0], ks);
  }
  uint32_t* counters =
      direct ? reinterpret_cast<uint32_t*>(d->stage[slot] + d->stage_cap[slot] - kStageTail)
             : nullptr;
  status = launch_mandel(ctx, d, dout, mt, chunks, prec, maxit, exact, px, ks, counters,
                         &batch[0]->actor->tune);
  if (direct) {
    ctx->st_direct++;
    ctx->st_d2h += px * 4;  // written to the replies by the kernel
  }
  phase(1);
  if (tev[0])
    cudaEventRecord(tev[1], ks);
  const double t_launched = trace_now_ms();
  // the reply segment table goes up on the compute stream: an upload-ring
  // slot recorded on the copy stream would only free up behind every queued
  // copy-out, and reusing it would block the dispatcher
  const bool inline_segs = segs.size() <= kInlineSegs;
  if (status == CAFXG_OK && px && all_pinned && !inline_segs && !direct) {
    size_t sb = segs.size() * sizeof(CopySeg);
    status = cuda_status(cudaMallocAsync((void**)&dsegs, sb, ks), "segs alloc");
    if (status == CAFXG_OK)
      status = upload(d, dsegs, segs.data(), sb, ks);
  }
  // the reply copy-out runs on the copy stream so it overlaps the next
  // batch's compute (a storm moves 16 KiB per request over PCIe; copying on
  // the compute stream instead was slower even for closed-loop trickles,
  // 144 -> 218 ms, because it serialises copy-out and the next kernel)
  cudaStream_t cs = direct ? ks : d->d2h;
  if (status == CAFXG_OK && px && !direct)
    status = stream_after_pooled(d, d->d2h, ks);
  phase(2);
  if (status == CAFXG_OK && px && !direct) {
    if (all_pinned) {
      {
        int e = inline_segs ? copy_segments_inline_launch(segs.data(), (uint32_t)segs.size(), cs)
                            : copy_segments_launch(dsegs, (uint32_t)segs.size(), cs);
        status = cuda_status((cudaError_t)e, "reply scatter launch");
        ctx->st_launches++;
      }
    } else {
      bounce = (uint32_t*)ctx->pinned.alloc(px * 4);
      if (!bounce)
        status = fail(CAFXG_E_CONFIG, "pinned bounce allocation failed");
      else
        status = cuda_status(cudaMemcpyAsync(bounce, dout, px * 4, cudaMemcpyDeviceToHost,
                                             cs), "batch download");
    }
    ctx->st_d2h += px * 4;
  }
  phase(3);
  if (dsegs)
    cudaFreeAsync(dsegs, cs);
  if (!direct)
    cudaEventRecord(d->stage_ev[slot], cs);  // slot free once the copy-out is done
  if (tev[0])
    cudaEventRecord(tev[2], cs);
  ctx->st_batches++;
  note_max_batch(ctx, batch.size());
  if (status != CAFXG_OK) {
    if (bounce)
      ctx->pinned.free(bounce);
    fail_all(status);
    return;
  }
  push_completion(ctx, d, cs,
                  [ctx, d, batch = std::move(batch), bounce, t_begin, t_lock, t_built,
                   t_launched, tev0 = tev[0], tev1 = tev[1], tev2 = tev[2],
                   t_sub = trace_now_ms()](int st) mutable {
                    const double t_done = trace_now_ms();
                    size_t n = batch.size();
                    finish_batch(ctx, std::move(batch), bounce, st);
                    if (trace_on())
                      fprintf(stderr,
                              "cafxg batch of %zu: build %.3f lock %.3f built %.3f "
                              "launched %.3f submit %.3f device-done %.3f "
                              "callbacks-handed-off %.3f ms\n",
                              n, t_begin, t_lock, t_built, t_launched, t_sub, t_done,
                              trace_now_ms());
                    if (tev0) {
                      float g[3] = {};
                      cudaEvent_t es[3] = {tev0, tev1, tev2};
                      for (int i = 0; i < 3; ++i) {
                        cudaEventElapsedTime(&g[i], d->trace_ref, es[i]);
                        cudaEventDestroy(es[i]);
                      }
                      fprintf(stderr,
                              "cafxg   gpu: kernel %.3f..%.3f copy-out done %.3f ms\n",
                              d->trace_ref_ms + g[0], d->trace_ref_ms + g[1],
                              d->trace_ref_ms + g[2]);
                    }
                  });
  phase(4);
}

Device* pick_device(cafxg_ctx* ctx) {
  // least in-flight work, round-robin among ties
  size_t n = ctx->devs.size();
  uint32_t start = ctx->rr.fetch_add(1);
  Device* best = nullptr;
  for (size_t i = 0; i < n; ++i) {
    Device* d = ctx->devs[(start + i) % n].get();
    if (!best || d->inflight.load() < best->inflight.load())
      best = d;
  }
  return best;
}

void dispatcher_loop(cafxg_ctx* ctx) {
  raise_priority();
  std::deque<Request*> queue;
  uint64_t queued_px = 0;
  // A trickle of requests (closed-loop clients) coalesces while kSoftInflight
  // batches run; a backlog of at least one full batch (open-loop bursts) may
  // fill the pipeline up to kMaxInflight.
  static const int soft = [] {  // CAFXG_SOFT_INFLIGHT: experiments only
    const char* e = getenv("CAFXG_SOFT_INFLIGHT");
    const int v = e ? atoi(e) : 0;
    return v > 0 && v <= kMaxInflight ? v : kSoftInflight;
  }();
  auto may_dispatch = [&](const Device* d) {
    const int n = d->inflight.load();
    return n < soft || (n < kMaxInflight && queued_px >= kMaxBatchPx);
  };
  while (true) {
    {
      std::unique_lock<std::mutex> lk(ctx->disp_mu);
      ctx->disp_cv.wait(lk, [&] {
        if (ctx->disp_stop)
          return true;
        if (ctx->inbox.load(std::memory_order_acquire) != nullptr && queue.empty())
          return true;
        if (!queue.empty()) {
          for (auto& d : ctx->devs)
            if (may_dispatch(d.get()))
              return true;
          return false;
        }
        return ctx->disp_wake;
      });
      ctx->disp_wake = false;
      if (ctx->disp_stop && queue.empty() && ctx->inbox.load() == nullptr)
        return;
    }
    // drain the inbox (LIFO stack) and append in FIFO order
    Request* head = ctx->inbox.exchange(nullptr, std::memory_order_acq_rel);
    std::vector<Request*> fresh;
    for (Request* r = head; r; r = r->next)
      fresh.push_back(r);
    for (auto it = fresh.rbegin(); it != fresh.rend(); ++it) {
      queue.push_back(*it);
      queued_px += (*it)->pixels;
    }
    if (queue.empty())
      continue;
    Device* d = pick_device(ctx);
    if (!may_dispatch(d) && !ctx->disp_stop)
      continue;  // wait for a completion; meanwhile the batch keeps growing
    // assemble one batch: leading requests of one kernel kind / precision
    std::vector<Request*> batch;
    uint64_t px = 0;
    while (!queue.empty()) {
      Request* r = queue.front();
      if (!r->actor->alive.load() || ctx->lost.load()) {
        queue.pop_front();
        queued_px -= r->pixels;
        push_completion(ctx, d, d->compute, [r](int) { finish_request(r, CAFXG_E_DOWN); });
        continue;
      }
      if (r->actor->kernel == Kernel::matrix_multiply) {
        if (!batch.empty())
          break;
        queue.pop_front();
        cafxg_sgemm_desc g{};
        g.M = g.N = g.K = (uint32_t)r->actor->dims[0];
        g.mode = r->actor->tune.sgemm_mode;
        g.splits = r->actor->tune.sgemm_splits;
        int s;
        try {
          s = sgemm_submit_impl(
              ctx, &g, r->a, r->b, (float*)r->out,
              [](void* u, int st) { finish_request((Request*)u, st); }, r);
        } catch (const std::exception& ex) {
          s = fail(CAFXG_E_CONFIG, "matrix_multiply: %s", ex.what());
        }
        if (s != CAFXG_OK)
          push_completion(ctx, d, d->compute, [r, s](int) { finish_request(r, s); });
        else
          ctx->st_requests--;  // counted by finish_request
        break;
      }
      if (!batch.empty() &&
          (r->precision != batch[0]->precision || !same_tuning(r->actor, batch[0]->actor) ||
           px + r->pixels > kMaxBatchPx))
        break;
      queue.pop_front();
      queued_px -= r->pixels;
      batch.push_back(r);
      px += r->pixels;
    }
    if (!batch.empty()) {
      if (trace_on())
        fprintf(stderr, "cafxg dispatch %.3f ms: batch %zu, %zu queued behind, inflight %d\n",
                trace_now_ms(), batch.size(), queue.size(), (int)d->inflight.load());
      const auto b0 = std::chrono::steady_clock::now();
      run_guarded("actor batch", [&] { run_mandel_batch(ctx, d, std::move(batch)); });
      ctx->st_batch_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                              std::chrono::steady_clock::now() - b0)
                              .count();
    }
  }
}

void wake_dispatcher(cafxg_ctx* ctx) {
  {
    std::lock_guard<std::mutex> lk(ctx->disp_mu);
    ctx->disp_wake = true;
  }
  ctx->disp_cv.notify_one();
}

}  // namespace cafxg

using namespace cafxg;

extern "C" {

// ---- actors --------------------------------------------------------------------

// The kernels' signatures, normalised like spawn_cl's template argument
// (PAPER.md:357-361): result type first, then the inputs.
static const char* kernel_signature(Kernel k) {
  return k == Kernel::matrix_multiply ? "f32*(f32*,f32*)" : "u32*(mandel_desc*)";
}

static int kernel_by_name(const char* name, Kernel* k) {
  if (!std::strcmp(name, "mandelbrot"))
    *k = Kernel::mandelbrot;
  else if (!std::strcmp(name, "matrix_multiply"))
    *k = Kernel::matrix_multiply;
  else
    return fail(CAFXG_E_UNKNOWN_TYPE, "spawn: no kernel named '%s'", name);
  return CAFXG_OK;
}

size_t cafxg_completion_batch(void) { return t_completion_batch; }

int cafxg_kernel_signature(const char* kernel_name, char* buf, size_t cap) {
  if (!kernel_name || !buf)
    return fail(CAFXG_E_CONFIG, "kernel_signature: null argument");
  Kernel k;
  CAFXG_TRY(kernel_by_name(kernel_name, &k));
  const char* sig = kernel_signature(k);
  if (std::strlen(sig) + 1 > cap)
    return fail(CAFXG_E_OUT_OF_RANGE, "kernel_signature: buffer of %zu bytes too small", cap);
  std::memcpy(buf, sig, std::strlen(sig) + 1);
  return CAFXG_OK;
}

static int validate_tuning(Kernel k, const cafxg_tuning& t) {
  for (uint32_t r : t.reserved)
    if (r)
      return fail(CAFXG_E_CONFIG, "tuning: reserved fields must be 0");
  if (k == Kernel::mandelbrot) {
    if (t.block_steps && (t.block_steps < 16 || t.block_steps > 64 || t.block_steps % 8))
      return fail(CAFXG_E_CONFIG, "tuning: block_steps must be 16..64 and a multiple of 8");
    if (t.sgemm_mode || t.sgemm_splits)
      return fail(CAFXG_E_CONFIG, "tuning: sgemm fields on a mandelbrot actor");
  } else {
    if (t.sgemm_mode > CAFXG_SGEMM_3XTF32)
      return fail(CAFXG_E_CONFIG, "tuning: bad sgemm_mode");
    if (t.sgemm_splits > 8 || (t.sgemm_splits & (t.sgemm_splits - 1)))
      return fail(CAFXG_E_CONFIG, "tuning: sgemm_splits must be 0, 1, 2, 4 or 8");
    if (t.block_steps || t.max_ctas)
      return fail(CAFXG_E_CONFIG, "tuning: mandelbrot fields on a matrix_multiply actor");
  }
  return CAFXG_OK;
}

int cafxg_spawn_ex(cafxg_ctx* ctx, const char* kernel_name, const char* signature,
                   const uint64_t* dims, size_t ndims, const cafxg_tuning* tuning,
                   cafxg_actor** out) try {
  if (!ctx || !kernel_name || !out)
    return fail(CAFXG_E_CONFIG, "spawn: null argument");
  *out = nullptr;
  Kernel k;
  CAFXG_TRY(kernel_by_name(kernel_name, &k));
  if (signature && std::strcmp(signature, kernel_signature(k)) != 0)
    return fail(CAFXG_E_INTERFACE_MISMATCH, "spawn_cl: signature %s does not match kernel %s %s",
                signature, kernel_name, kernel_signature(k));
  if (k == Kernel::matrix_multiply) {
    // spawn_cl<float*(float*,float*)>(src, "matrix_multiply", {size, size})
    if (ndims != 2 || !dims || dims[0] == 0 || dims[0] != dims[1] || dims[0] > (1u << 16))
      return fail(CAFXG_E_INTERFACE_MISMATCH,
                  "spawn: matrix_multiply takes dims {size, size}");
  }
  cafxg_tuning t{};
  if (tuning) {
    CAFXG_TRY(validate_tuning(k, *tuning));
    t = *tuning;
  }
  auto* a = new cafxg_actor;
  a->ctx = ctx;
  a->kernel = k;
  a->ndims = std::min<size_t>(ndims, 3);
  for (size_t i = 0; i < a->ndims; ++i)
    a->dims[i] = dims[i];
  a->tune = t;
  *out = a;
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_spawn_ex: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_spawn_ex: unknown exception");
}

int cafxg_spawn(cafxg_ctx* ctx, const char* kernel_name, const uint64_t* dims, size_t ndims,
                cafxg_actor** out) {
  return cafxg_spawn_ex(ctx, kernel_name, nullptr, dims, ndims, nullptr, out);
}

int actor_check(cafxg_actor* a, const void* const* in, const size_t* in_bytes,
                       size_t n_in, size_t* reply_bytes) {
  if (!a)
    return fail(CAFXG_E_CONFIG, "enqueue: null actor");
  if (n_in && (!in || !in_bytes))
    return fail(CAFXG_E_CONFIG, "enqueue: null inputs");
  if (a->kernel == Kernel::mandelbrot) {
    if (n_in != 1)
      return fail(CAFXG_E_INTERFACE_MISMATCH, "mandelbrot takes one descriptor buffer");
    if (in_bytes[0] == 0 || in_bytes[0] % sizeof(cafxg_mandel_desc) != 0 || !in[0])
      return fail(CAFXG_E_TYPE_MISMATCH,
                  "mandelbrot input must hold whole cafxg_mandel_desc records");
    const auto* t = static_cast<const cafxg_mandel_desc*>(in[0]);
    size_t n = in_bytes[0] / sizeof(cafxg_mandel_desc);
    uint64_t px = 0;
    int prec = t[0].precision;
    for (size_t i = 0; i < n; ++i) {
      CAFXG_TRY(validate_mandel(t[i]));
      if ((int)t[i].precision != prec)
        return fail(CAFXG_E_CONFIG, "mandelbrot: one precision per request");
      px += (uint64_t)t[i].nrows * t[i].ncols;
    }
    if (px == 0)
      return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot: request without pixels");
    *reply_bytes = px * 4;
    return CAFXG_OK;
  }
  size_t sz = a->dims[0];
  size_t mb = sz * sz * sizeof(float);
  if (n_in != 2)
    return fail(CAFXG_E_INTERFACE_MISMATCH, "matrix_multiply takes (matrix1, matrix2)");
  if (in_bytes[0] != mb || in_bytes[1] != mb || !in[0] || !in[1])
    return fail(CAFXG_E_TYPE_MISMATCH, "matrix_multiply inputs must be size*size floats");
  *reply_bytes = mb;
  return CAFXG_OK;
}

size_t cafxg_actor_reply_bytes(cafxg_actor* a, const void* const* in, const size_t* in_bytes,
                               size_t n_in) {
  size_t rb = 0;
  return actor_check(a, in, in_bytes, n_in, &rb) == CAFXG_OK ? rb : 0;
}

int cafxg_actor_enqueue(cafxg_actor* a, const void* const* in, const size_t* in_bytes,
                        size_t n_in, void* out, size_t out_bytes, cafxg_done_fn done,
                        void* user) try {
  size_t rb = 0;
  CAFXG_TRY(actor_check(a, in, in_bytes, n_in, &rb));
  if (!a->alive.load())
    return fail(CAFXG_E_DOWN, "enqueue: actor terminated");
  CAFXG_TRY(check_alive(a->ctx));
  if (!out || out_bytes != rb)
    return fail(CAFXG_E_TYPE_MISMATCH, "enqueue: reply buffer must be %zu bytes", rb);
  auto* r = new Request;
  r->actor = a;
  r->out = out;
  r->out_bytes = out_bytes;
  r->done = done;
  r->user = user;
  if (a->kernel == Kernel::mandelbrot) {
    const auto* t = static_cast<const cafxg_mandel_desc*>(in[0]);
    size_t n = in_bytes[0] / sizeof(cafxg_mandel_desc);
    r->tile0 = t[0];
    if (n > 1)
      r->more.assign(t + 1, t + n);
    r->ntiles = (uint32_t)n;
    r->precision = (int)t[0].precision;
    uint64_t off = 0;
    for (size_t k = 0; k < n; ++k) {
      cafxg_mandel_desc& x = k == 0 ? r->tile0 : r->more[k - 1];
      x.out_offset = off;  // tiles packed in order in the reply
      off += (uint64_t)x.nrows * x.ncols;
      r->max_iter = std::max(r->max_iter, x.max_iter);
      r->exact = r->exact || use_exact(a->ctx, x);
    }
    r->pixels = off;
    // classified on the client's thread so the dispatcher stays lean
    r->out_pinned = a->ctx->pinned.contains(out, out_bytes) || host_is_pinned(out, out_bytes);
  } else {
    r->a = static_cast<const float*>(in[0]);
    r->b = static_cast<const float*>(in[1]);
  }
  a->refs.fetch_add(1);
  a->pending.fetch_add(1);
  cafxg_ctx* ctx = a->ctx;
  ctx->actor_open.fetch_add(1);
  if (a->kernel == Kernel::mandelbrot && r->pixels >= kLargeActorPx) {
    // a large request is never batched: submitted from the caller's thread
    // straight into the host-request path (row bands over every device,
    // overlapped waves), which saves the dispatcher hop (~10 us of a 0.2 ms
    // cfg1 request); non-blocking like the inbox
    int s;
    try {
      std::vector<cafxg_mandel_desc> tiles(r->ntiles);
      for (uint32_t k = 0; k < r->ntiles; ++k)
        tiles[k] = r->tile(k);
      s = mandel_submit_impl(
          ctx, tiles.data(), tiles.size(), static_cast<uint32_t*>(r->out),
          [](void* u, int st) { finish_request((Request*)u, st); }, r, &a->tune);
    } catch (const std::exception& ex) {
      s = fail(CAFXG_E_CONFIG, "enqueue: %s", ex.what());
    }
    if (s != CAFXG_OK) {
      std::string err = t_last_error;
      Device* d = ctx->devs[0].get();
      std::lock_guard<std::mutex> g(d->submit_mu);
      push_completion(ctx, d, d->compute, [r, s](int) { finish_request(r, s); });
      t_last_error = err;
    } else {
      ctx->st_requests--;  // counted by finish_request
    }
    return CAFXG_OK;
  }
  Request* head = ctx->inbox.load(std::memory_order_relaxed);
  do {
    r->next = head;
  } while (!ctx->inbox.compare_exchange_weak(head, r, std::memory_order_release,
                                             std::memory_order_relaxed));
  if (head == nullptr)  // empty -> non-empty: the dispatcher may sleep
    wake_dispatcher(ctx);
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_actor_enqueue: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_actor_enqueue: unknown exception");
}

int cafxg_actor_quit(cafxg_actor* a) {
  if (!a)
    return fail(CAFXG_E_CONFIG, "quit: null actor");
  a->alive.store(false);
  wake_dispatcher(a->ctx);
  return CAFXG_OK;
}

int cafxg_actor_release(cafxg_actor* a) {
  if (!a)
    return CAFXG_OK;
  a->alive.store(false);
  wake_dispatcher(a->ctx);
  actor_unref(a);
  return CAFXG_OK;
}

}  // extern "C"
