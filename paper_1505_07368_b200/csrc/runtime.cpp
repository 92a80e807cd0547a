// libcafxg.so host runtime: contexts, devices, pinned pool, completion
// threads, multi-device request splitting, compute actors and the batching
// dispatcher behind the C ABI of include/cafxg.h.
//
// Reference mapping (what each piece replaces in CAF's OpenCL path):
//  * cafxg_spawn / cafxg_actor_enqueue  -> spawn_cl + the actor's enqueue
//    (seam abstract_actor::enqueue, abstract_actor.hpp:36);
//  * completion threads                 -> the reply path of local_actor::
//    respond (local_actor.cpp:319-329), run off the scheduler workers;
//  * the dispatcher's MPSC inbox        -> cached_stack_mailbox
//    (mailbox.cpp:13-62): one CAS per enqueue, one exchange per drain;
//  * cafxg_actor_quit                   -> hard-kill exit + request_down
//    errors for pending requests (actor_system.cpp:243-258,
//    abstract_actor.cpp:126-131).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.hpp"
#include "mandelbrot.cuh"
#include "sgemm.cuh"

namespace cafxg {

// ---- error context -----------------------------------------------------------

static thread_local std::string t_last_error;

void set_last_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_last_error = buf;
}

void clear_last_error() { t_last_error.clear(); }

// ---- pinned host pool -----------------------------------------------------------
// Page-locked, portable, device-mapped buffers cached by power-of-two size
// class. Reply buffers that live here are written by DMA or by the reply
// scatter kernel directly.
class PinnedPool {
 public:
  ~PinnedPool() {
    std::lock_guard<std::mutex> g(mu_);
    for (auto& kv : free_)
      for (void* p : kv.second)
        cudaFreeHost(p);
    for (auto& kv : live_)
      cudaFreeHost(kv.first);
  }

  void* alloc(size_t bytes) {
    size_t cls = size_class(bytes);
    {
      std::lock_guard<std::mutex> g(mu_);
      auto it = free_.find(cls);
      if (it != free_.end() && !it->second.empty()) {
        void* p = it->second.back();
        it->second.pop_back();
        live_[p] = cls;
        return p;
      }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, cls, cudaHostAllocPortable | cudaHostAllocMapped) !=
        cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    std::lock_guard<std::mutex> g(mu_);
    live_[p] = cls;
    {
      std::unique_lock<std::shared_mutex> w(ranges_mu_);
      ranges_[(uintptr_t)p] = cls;
    }
    return p;
  }

  bool free(void* p) {
    std::lock_guard<std::mutex> g(mu_);
    auto it = live_.find(p);
    if (it == live_.end())
      return false;
    free_[it->second].push_back(p);
    live_.erase(it);
    return true;
  }

  // [p, p+bytes) inside one pool buffer (no driver call). Every client
  // thread classifies its reply buffer here, so the common case takes no lock
  // at all: a thread-local cache of the last buffer hit (pool buffers stay
  // pinned and device-mapped until the context closes, so a cached range
  // never goes stale, and a buffer on the free list still qualifies);
  // otherwise a shared (reader) lock on the range map.
  bool contains(const void* p, size_t bytes) const {
    struct Hit {
      uint64_t pool = 0;
      uintptr_t base = 0;
      size_t size = 0;
    };
    thread_local Hit hit;
    const uintptr_t a = (uintptr_t)p;
    if (hit.pool == id_ && a >= hit.base && a + bytes <= hit.base + hit.size)
      return true;
    std::shared_lock<std::shared_mutex> r(ranges_mu_);
    auto it = ranges_.upper_bound(a);
    if (it == ranges_.begin())
      return false;
    --it;
    if (a + bytes > it->first + it->second)
      return false;
    hit = Hit{id_, it->first, it->second};
    return true;
  }

 private:
  static size_t size_class(size_t bytes) {
    size_t c = 4096;
    while (c < bytes)
      c <<= 1;
    return c;
  }
  std::mutex mu_;
  std::unordered_map<void*, size_t> live_;
  std::map<size_t, std::vector<void*>> free_;
  mutable std::shared_mutex ranges_mu_;
  std::map<uintptr_t, size_t> ranges_;  // every buffer ever allocated
  // unique per pool instance (never reused), so a thread-local cache entry of
  // a closed context can never match a later one
  static inline std::atomic<uint64_t> next_id_{1};
  const uint64_t id_ = next_id_.fetch_add(1);
};

// True when [p, p+bytes) is page-locked host memory the device can address
// (our pool, cudaHostRegister'ed or torch pin_memory buffers).
static bool host_is_pinned(const void* p, size_t bytes) {
  if (!p)
    return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type != cudaMemoryTypeHost || a.devicePointer != p)
    return false;
  if (bytes > 1) {
    cudaPointerAttributes b{};
    const char* last = static_cast<const char*>(p) + bytes - 1;
    if (cudaPointerGetAttributes(&b, last) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return b.type == cudaMemoryTypeHost && b.devicePointer == last;
  }
  return true;
}

// ---- NCCL (loaded lazily; only multi-device sgemm needs it) ------------------------

struct NcclApi {
  bool ok = false;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  bool load() {
    if (ok)
      return true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h)
      h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h)
      return false;
    CommInitAll = (decltype(CommInitAll))dlsym(h, "ncclCommInitAll");
    AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
    GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    ok = CommInitAll && AllGather && GroupStart && GroupEnd && CommDestroy;
    return ok;
  }
};

// ---- devices and completion -----------------------------------------------------------

struct Completion {
  cudaEvent_t ev;
  std::function<void(int)> fn;
};

constexpr uint32_t kSchedSlots = 1024;
// Actor batching: at most kMaxInflight batches per device before the
// dispatcher holds (arrivals meanwhile coalesce into the next batch), each of
// at most kMaxBatchPx pixels (a single larger request is its own batch).
// Batches are kept small enough that the reply copy-out of one overlaps the
// kernel of the next and the pipeline drains quickly after the last request.
constexpr int kMaxInflight = 8;
constexpr int kSoftInflight = 4;
// Staging slot tail: the direct-reply tile counters (kInlineTiles u32).
constexpr size_t kStageTail = 256;
// Direct reply: per-tile limit (one warp copies the finished tile: 16 KiB
// storm tiles take 32 rounds of 16-byte stores; a 1M-pixel band would stall
// its warp for milliseconds).
constexpr uint64_t kDirectTilePx = 64u << 10;
// Launches of at most this many pixels compute coordinates inline (one fp64
// divide per pixel start) instead of through a coordinate-table launch and
// its allocation: for cfg1's 512K-pixel first wave the table path cost ~8 us
// of host issue time before the escape kernel could start.
constexpr uint64_t kInlineCoordsPx = 4u << 20;
constexpr uint64_t kInlineCopyPx = 256u << 10;  // copy-out on the compute stream below  // beyond this only when a full batch is queued
constexpr uint64_t kMaxBatchPx = 16ull << 20;
constexpr int kUpSlots = 16;
constexpr size_t kUpSlotBytes = 2u << 20;

struct Device {
  int ordinal = 0;
  int sms = 0;
  cudaStream_t compute = nullptr, d2h = nullptr, h2d = nullptr;
  // second compute stream: consecutive waves of a host request alternate
  // between the two, so a wave's kernel fills the SMs the previous wave's
  // tail leaves idle
  cudaStream_t compute2 = nullptr;
  uint32_t* sched = nullptr;  // kSchedSlots x {cursor, finished}
  std::atomic<uint32_t> sched_next{0};
  std::mutex submit_mu;

  std::mutex cq_mu;
  std::condition_variable cq_cv;
  std::deque<Completion> cq;
  std::vector<cudaEvent_t> ev_free;
  bool stop = false;
  std::thread completer;
  std::atomic<int> inflight{0};
  int mandel_occ[2][8][2][2] = {};  // see mandel_cfg
  // pinned staging ring for descriptor uploads (a pageable cudaMemcpyAsync
  // may wait for earlier work on the stream, serialising host and device)
  std::mutex up_mu;
  uint8_t* up_base = nullptr;
  cudaEvent_t up_ev[16] = {};
  bool up_armed[16] = {};
  uint32_t up_next = 0;
  // batch staging ring (actor batches): one device buffer per in-flight
  // batch, reused in order. A fresh cudaMallocAsync per batch can block the
  // dispatcher while the pool grows; this ring grows only in warm-up. Reuse
  // of slot i waits (on the device) for the copy-out that last read it.
  uint8_t* stage[kMaxInflight] = {};
  size_t stage_cap[kMaxInflight] = {};
  cudaEvent_t stage_ev[kMaxInflight] = {};
  bool stage_on_copy[kMaxInflight] = {};  // last user recorded stage_ev on d2h
  uint32_t stage_next = 0;
  // reusable events for host request pipelines (caller holds submit_mu): an
  // event may be re-recorded as soon as the waits on its last record are
  // enqueued, so these never need to be destroyed per request
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t order_ev = nullptr;   // stream_after_pooled
  // grow-only workspace of the host sgemm row-block pipeline (caller holds
  // submit_mu; each request orders itself after the previous one's use)
  float* sgemm_ws = nullptr;
  size_t sgemm_ws_bytes = 0;
  cudaEvent_t trace_ref = nullptr;  // CAFXG_TRACE time base
  double trace_ref_ms = 0;

  uint32_t* next_sched() {
    uint32_t i = sched_next.fetch_add(1, std::memory_order_relaxed) % kSchedSlots;
    return sched + 2 * i;
  }
};

}  // namespace cafxg

using namespace cafxg;

struct Request;

struct cafxg_ctx {
  std::vector<std::unique_ptr<Device>> devs;
  PinnedPool pinned;
  // outstanding completion records (cafxg_sync)
  std::mutex sync_mu;
  std::condition_variable sync_cv;
  uint64_t submitted = 0, completed = 0;
  // statistics
  std::atomic<uint64_t> st_requests{0}, st_batches{0}, st_launches{0},
      st_h2d{0}, st_d2h{0}, st_max_batch{0};
  std::atomic<uint64_t> st_batch_ns{0};  // dispatcher time spent submitting batches
  std::atomic<uint64_t> st_direct{0};    // batches replied by the escape kernel itself
  std::atomic<uint64_t> st_phase_ns[6] = {};  // run_mandel_batch phases (CAFXG_STATS)
  // actor dispatcher
  std::atomic<Request*> inbox{nullptr};
  std::mutex disp_mu;
  std::condition_variable disp_cv;
  bool disp_stop = false;
  bool disp_wake = false;
  std::thread dispatcher;
  std::atomic<uint32_t> rr{0};
  std::atomic<uint64_t> actor_open{0};  // enqueued, not yet completed
  // reply-callback threads (finish_batch)
  std::mutex cb_mu;
  std::condition_variable cb_cv;
  std::deque<std::function<void()>> cb_q;
  bool cb_stop = false;
  std::vector<std::thread> cb_threads;
  bool force_exact = false;  // CAFXG_EXACT_STEP=1: always the 8-op step
  // CAFXG_VIRTUAL_DEVICES=V: V context devices on one physical GPU (own
  // streams, scheduler ring and completion thread each) so the multi-device
  // split/join logic runs on a single-GPU box; B is then replicated by
  // device-to-device copies instead of NCCL (which rejects duplicate GPUs)
  bool virtual_devs = false;
  // NCCL communicators for multi-device sgemm (one per device)
  std::mutex nccl_mu;
  bool nccl_failed = false;
  NcclApi nccl;
  std::vector<ncclComm_t> comms;
};

namespace cafxg {

// Host clock for CAFXG_TRACE timelines (ms since first use).
static double trace_now_ms() {
  static const auto t0 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

static void note_max_batch(cafxg_ctx* ctx, uint64_t n) {
  uint64_t cur = ctx->st_max_batch.load();
  while (n > cur && !ctx->st_max_batch.compare_exchange_weak(cur, n)) {
  }
}

// Backend threads (dispatcher, completion) get a higher scheduling weight
// than client threads when the process may raise it (best effort): under a
// request storm, clients outnumber cores, and a starved completion thread
// leaves the device idle with finished batches counted as in flight.
static void raise_priority() {
  setpriority(PRIO_PROCESS, (id_t)syscall(SYS_gettid), -10);
}

static void completion_loop(cafxg_ctx* ctx, Device* d) {
  raise_priority();
  cudaSetDevice(d->ordinal);
  while (true) {
    Completion c;
    {
      std::unique_lock<std::mutex> lk(d->cq_mu);
      d->cq_cv.wait(lk, [&] { return d->stop || !d->cq.empty(); });
      if (d->cq.empty())
        return;
      c = std::move(d->cq.front());
      d->cq.pop_front();
    }
    cudaError_t e = cudaEventSynchronize(c.ev);
    int status = CAFXG_OK;
    if (e != cudaSuccess)
      status = cuda_status(e, "device work failed");
    c.fn(status);
    {
      std::lock_guard<std::mutex> lk(d->cq_mu);
      d->ev_free.push_back(c.ev);
    }
    d->inflight.fetch_sub(1);
    {
      std::lock_guard<std::mutex> lk(ctx->sync_mu);
      ++ctx->completed;
    }
    ctx->sync_cv.notify_all();
    ctx->disp_cv.notify_all();
  }
}

// Records an event on `stream` and hands `fn` to the device's completion
// thread. Caller holds d->submit_mu (so records stay in stream order).
static int push_completion(cafxg_ctx* ctx, Device* d, cudaStream_t stream,
                           std::function<void(int)> fn) {
  cudaEvent_t ev = nullptr;
  {
    std::lock_guard<std::mutex> lk(d->cq_mu);
    if (!d->ev_free.empty()) {
      ev = d->ev_free.back();
      d->ev_free.pop_back();
    }
  }
  if (!ev)
    CAFXG_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CAFXG_CUDA_TRY(cudaEventRecord(ev, stream));
  {
    std::lock_guard<std::mutex> lk(ctx->sync_mu);
    ++ctx->submitted;
  }
  d->inflight.fetch_add(1);
  {
    std::lock_guard<std::mutex> lk(d->cq_mu);
    d->cq.push_back(Completion{ev, std::move(fn)});
  }
  d->cq_cv.notify_one();
  return CAFXG_OK;
}

// Host -> device copy of small descriptor arrays through the device's pinned
// staging ring, so the call never waits for earlier work on `stream`.
static int upload(Device* d, void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (bytes > kUpSlotBytes)
    return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream),
                       "descriptor upload");
  std::lock_guard<std::mutex> g(d->up_mu);
  uint32_t i = d->up_next++ % kUpSlots;
  if (d->up_armed[i])
    CAFXG_CUDA_TRY(cudaEventSynchronize(d->up_ev[i]));
  uint8_t* p = d->up_base + (size_t)i * kUpSlotBytes;
  std::memcpy(p, src, bytes);
  CAFXG_CUDA_TRY(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, stream));
  CAFXG_CUDA_TRY(cudaEventRecord(d->up_ev[i], stream));
  d->up_armed[i] = true;
  return CAFXG_OK;
}

// Joins the per-device parts of one request; the last part reports.
struct Join {
  std::atomic<int> remaining{0};
  std::atomic<int> status{CAFXG_OK};
  cafxg_done_fn done = nullptr;
  void* user = nullptr;
  std::function<void()> on_ok;  // runs before done when every part succeeded

  void part_done(int s) {
    if (s != CAFXG_OK) {
      int expected = CAFXG_OK;
      status.compare_exchange_strong(expected, s);
    }
    if (remaining.fetch_sub(1) == 1) {
      int st = status.load();
      if (st == CAFXG_OK && on_ok)
        on_ok();
      if (done)
        done(user, st);
      delete this;
    }
  }
};

// ---- Mandelbrot planning -----------------------------------------------------------

static int validate_mandel(const cafxg_mandel_desc& t) {
  if (!std::isfinite(t.x0) || !std::isfinite(t.x1) || !std::isfinite(t.y0) ||
      !std::isfinite(t.y1))
    return fail(CAFXG_E_CONFIG, "mandelbrot: region must be finite");
  if (t.width == 0 || t.height == 0)
    return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot: empty image");
  if ((uint64_t)t.row0 + t.nrows > t.height || (uint64_t)t.col0 + t.ncols > t.width)
    return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot: tile outside the image");
  if (t.precision > 1 || t.sampling > 1)
    return fail(CAFXG_E_CONFIG, "mandelbrot: bad precision or sampling");
  if (t.max_iter > (1u << 30))
    return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot: max_iter above 2^30");
  if ((uint64_t)t.nrows * t.ncols > 0xffffffffull)
    return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot: tile above 2^32 pixels");
  return CAFXG_OK;
}

static double coord(double lo, double hi, uint32_t i, uint32_t n, double s) {
  volatile double k = (double)i + s;  // volatile: keep every rounding explicit
  volatile double p = k * (hi - lo);
  volatile double q = p / (double)n;
  return lo + q;
}

// Smallest nonzero |ci| the tile's rows produce, in the request precision.
// The map row -> ci is monotone, so the minimum sits next to the zero
// crossing or at an end row.
static double min_abs_ci(const cafxg_mandel_desc& t) {
  double s = t.sampling ? 0.5 : 0.0;
  int64_t cand[8] = {(int64_t)t.row0, (int64_t)t.row0 + t.nrows - 1};
  int nc = 2;
  double span = t.y1 - t.y0;
  if (span != 0.0) {
    double r = -t.y0 * (double)t.height / span - s;
    if (std::isfinite(r) && std::fabs(r) < 9.0e18) {
      for (int64_t k = (int64_t)std::floor(r) - 2; k <= (int64_t)std::floor(r) + 3; ++k)
        cand[nc++] = k;
    }
  }
  double best = INFINITY;
  for (int i = 0; i < nc; ++i) {
    const int64_t r = cand[i];
    if (r < (int64_t)t.row0 || r >= (int64_t)t.row0 + t.nrows)
      continue;
    double ci = coord(t.y0, t.y1, (uint32_t)r, t.height, s);
    double v = t.precision ? std::fabs(ci) : std::fabs((double)(float)ci);
    if (v > 0.0 && v < best)
      best = v;
  }
  return best;
}

// The 7-op escape step is bit-identical unless a row has a tiny nonzero ci
// (DESIGN.md §3): fp32 needs |ci| >= 2^-100, fp64 |ci| >= 2^-960.
static bool needs_exact_step(const cafxg_mandel_desc& t);
static bool use_exact(cafxg_ctx* ctx, const cafxg_mandel_desc& t) {
  return ctx->force_exact || needs_exact_step(t);
}
static bool needs_exact_step(const cafxg_mandel_desc& t) {
  double lim = t.precision ? std::ldexp(1.0, -960) : std::ldexp(1.0, -100);
  return min_abs_ci(t) < lim;
}

struct SubTile {
  cafxg_mandel_desc d;  // row0/nrows narrowed; out_offset = host offset
  uint64_t pixels;
};

// Work chunks of a tile: rows x ceil(ncols / chunk) (chunks never straddle
// rows, see mandel_kernel); a chunk is one refill generation of a warp.
static uint32_t tile_chunks(uint32_t nrows, uint32_t ncols, uint32_t precision) {
  const uint32_t c = chunk_px((int)precision);
  return nrows * ((ncols + c - 1) / c);
}

static void fill_mtile(MTile& m, const cafxg_mandel_desc& d, uint64_t out_off,
                       uint32_t chunk_begin) {
  m.x0 = d.x0;
  m.xspan = d.x1 - d.x0;
  m.y0 = d.y0;
  m.yspan = d.y1 - d.y0;
  m.s = d.sampling ? 0.5 : 0.0;
  m.width = d.width;
  m.height = d.height;
  m.row0 = d.row0;
  m.col0 = d.col0;
  m.nrows = d.nrows;
  m.ncols = d.ncols;
  m.max_iter = d.max_iter;
  m.chunk_begin = chunk_begin;
  m.chunks_per_row = (d.ncols + chunk_px((int)d.precision) - 1) / chunk_px((int)d.precision);
  m.out_off = (uint32_t)out_off;
  m.cx = m.cy = nullptr;
  m.reply = nullptr;
}

// Precondition of the deferred escape test (mandel_deferred_kernel): the
// tile's coordinate box stays outside the annulus 2 - 2^-10 < |c| < 2 + 2^-10,
// where an orbit could pass the reference's test and fall back below it.
static bool deferred_safe(const MTile& t) {
  auto at = [](double lo, double span, double s, uint32_t i, uint32_t n) {
    return lo + (((double)i + s) * span) / n;
  };
  double xa = at(t.x0, t.xspan, t.s, t.col0, t.width);
  double xb = at(t.x0, t.xspan, t.s, t.col0 + t.ncols - 1, t.width);
  double ya = at(t.y0, t.yspan, t.s, t.row0, t.height);
  double yb = at(t.y0, t.yspan, t.s, t.row0 + t.nrows - 1, t.height);
  if (xa > xb) std::swap(xa, xb);
  if (ya > yb) std::swap(ya, yb);
  const double dx = xa > 0 ? xa : (xb < 0 ? -xb : 0.0);
  const double dy = ya > 0 ? ya : (yb < 0 ? -yb : 0.0);
  const double rmin = std::hypot(dx, dy);
  const double rmax = std::hypot(std::max(std::fabs(xa), std::fabs(xb)),
                                 std::max(std::fabs(ya), std::fabs(yb)));
  const double eta = std::ldexp(1.0, -10), pad = 1e-6;  // pad: fp32 rounding of c
  return rmax < 2.0 - eta - pad || rmin > 2.0 + eta + pad;
}

// CAFXG_DIRECT_REPLY=0 keeps every batch on the reply-scatter launch
static bool direct_reply_enabled() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_DIRECT_REPLY");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CAFXG_DEFERRED=0 forces the per-step-checked kernel everywhere
static bool deferred_enabled() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_DEFERRED");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Unchecked block length B of the deferred kernel. Modelled cost per pixel
// that never escapes, relative to max_iter steps:
//   ceil(max_iter / B) * B / max_iter * (1 + alpha / B) + gamma * B
// (overshoot past max_iter; block-end test and refill, ~alpha steps' worth;
// replays of escaped blocks grow with B). alpha = 7 (fp32) / 2 (fp64: the
// steps cost twice as much) and gamma = 0.002 fit the block-length sweep
// (DESIGN.md §3.1): cfg3 (fp32, max_iter 1000) runs 38.0 / 35.7 / 35.2 /
// 34.9 / 35.0 ms at B = 32 / 40 / 48 / 56 / 64 and picks 56; the fp64
// reference mode (max_iter 500) picks 24. Each B is one fully unrolled PTX
// block (8-step units in a runtime loop were 5% slower at B = 32).
// CAFXG_BLOCK=<B> forces a length (multiple of 8; 16..64 unrolled).
static void pick_block(uint32_t max_iter, int precision, MandelLaunchCfg& c) {
  static const int env = [] {
    const char* e = getenv("CAFXG_BLOCK");
    return e ? atoi(e) : 0;
  }();
  auto set = [&](uint32_t b) {
    if (b >= 16 && b <= 64 && b % 8 == 0) {
      c.unit = (int)b;
      c.reps = 1;
    } else {
      c.unit = 8;
      c.reps = (int)(b / 8);
    }
  };
  if (env >= 8 && env % 8 == 0) {
    set((uint32_t)env);
    return;
  }
  const double alpha = precision ? 2.0 : 7.0, gamma = 0.002;
  uint32_t best = 32;
  double best_cost = 1e300;
  for (uint32_t b = 16; b <= 64; b += 8) {
    const double over = (double)((max_iter + b - 1) / b * b) / max_iter;
    const double cost = over * (1.0 + alpha / b) + gamma * b;
    if (cost < best_cost) {
      best = b;
      best_cost = cost;
    }
  }
  set(best);
}

static MandelLaunchCfg mandel_cfg(Device* d, int precision, uint32_t max_iter,
                                  bool exact, bool safe, uint64_t pixels) {
  MandelLaunchCfg c;
  // checked kernel: steps between votes (cfg1, max_iter 100: 16 steps 0.065 ms, 4 steps 0.074)
  c.ksteps = max_iter >= 512 ? 32 : max_iter >= 64 ? 16 : 4;
  static const int ks_env = [] {  // CAFXG_KSTEPS=4|16|32: experiments only
    const char* e = getenv("CAFXG_KSTEPS");
    return e ? atoi(e) : 0;
  }();
  if (ks_env == 4 || ks_env == 16 || ks_env == 32)
    c.ksteps = ks_env;
  c.exact = exact;
  c.deferred = safe && max_iter >= 256 && deferred_enabled();
  if (c.deferred)
    pick_block(max_iter, precision, c);
  // occupancy per kernel variant: [precision][checked ksteps 4/16/32 |
  // deferred unit 8/32][exact][deferred]
  const int vi = c.deferred ? c.unit / 8 - 1 : (c.ksteps == 4 ? 0 : c.ksteps == 16 ? 1 : 2);
  int& occ = d->mandel_occ[precision][vi][exact][c.deferred];
  if (occ == 0)
    occ = std::max(1, mandel_max_blocks_per_sm(precision, c.ksteps, exact, c.deferred,
                                               c.unit));
  const uint64_t per_block = (uint64_t)kMandelThreads * mandel_slots_per_thread(precision);
  uint64_t want = (pixels + per_block - 1) / per_block;
  uint64_t full = (uint64_t)d->sms * occ;
  c.grid = (int)std::max<uint64_t>(1, std::min(want, full));
  return c;
}

// Enqueues the Mandelbrot launches for `tiles` (all the same precision) on
// `stream`: one coordinate-table launch, then one escape launch per distinct
// max_iter (the kernel keeps max_iter launch-uniform). Descriptors beyond the
// inline capacity are uploaded first.
static int launch_mandel_group(cafxg_ctx* ctx, Device* d, uint32_t* out_base,
                               std::vector<MTile>& tiles, int precision, bool exact,
                               cudaStream_t stream, bool coords_only, bool skip_coords,
                               uint32_t* direct_counters = nullptr);

static int launch_mandel(cafxg_ctx* ctx, Device* d, uint32_t* out_base,
                         const std::vector<MTile>& tiles_in, uint32_t total_chunks,
                         int precision, uint32_t max_iter, bool exact,
                         uint64_t pixels, cudaStream_t stream,
                         uint32_t* direct_counters = nullptr) {
  (void)max_iter;
  if (total_chunks == 0)
    return CAFXG_OK;
  // coordinate tables (one column and one row table per tile) pay off for
  // big tiles; batches of small tiles (request storms) compute coordinates
  // inline in the escape kernel and save the table launch
  std::vector<MTile> tiles = tiles_in;
  // (and so do launches of few pixels in all: kInlineCoordsPx)
  bool small_tiles = true;
  for (auto& t : tiles)
    small_tiles = small_tiles && (uint64_t)t.ncols * t.nrows <= (64u << 10);
  const bool small = small_tiles || pixels <= kInlineCoordsPx;
  uint8_t* coords = nullptr;
  if (!small) {
    const size_t esz = precision ? sizeof(double) : sizeof(float);
    uint64_t ncoord = 0;
    for (auto& t : tiles)
      ncoord += (uint64_t)t.ncols + t.nrows;
    CAFXG_CUDA_TRY(cudaMallocAsync((void**)&coords, ncoord * esz + 16, stream));
    uint64_t off = 0;
    for (auto& t : tiles) {
      t.cx = coords + off * esz;
      t.cy = coords + (off + t.ncols) * esz;
      off += (uint64_t)t.ncols + t.nrows;
    }
    CAFXG_TRY(
        launch_mandel_group(ctx, d, out_base, tiles, precision, exact, stream, true, false));
  } else {
    for (auto& t : tiles)
      t.cx = t.cy = nullptr;
  }
  // group by max_iter (stable), re-basing the chunk numbering per group
  std::vector<uint32_t> its;
  for (auto& t : tiles)
    if (std::find(its.begin(), its.end(), t.max_iter) == its.end())
      its.push_back(t.max_iter);
  for (uint32_t it : its) {
    std::vector<MTile> grp;
    for (auto& t : tiles)
      if (t.max_iter == it)
        grp.push_back(t);
    if (direct_counters && its.size() != 1)
      return fail(CAFXG_E_CONFIG, "internal: direct reply across max_iter groups");
    CAFXG_TRY(launch_mandel_group(ctx, d, out_base, grp, precision, exact, stream, false, true,
                                  direct_counters));
  }
  if (coords)
    CAFXG_CUDA_TRY(cudaFreeAsync(coords, stream));
  return CAFXG_OK;
}

static int launch_mandel_group(cafxg_ctx* ctx, Device* d, uint32_t* out_base,
                               std::vector<MTile>& tiles, int precision, bool exact,
                               cudaStream_t stream, bool coords_only, bool skip_coords,
                               uint32_t* direct_counters) {
  uint32_t chunks = 0, max_extent = 0;
  uint64_t pixels = 0;
  for (auto& t : tiles) {
    t.chunk_begin = chunks;
    chunks += tile_chunks(t.nrows, t.ncols, (uint32_t)precision);
    pixels += (uint64_t)t.nrows * t.ncols;
    max_extent = std::max(max_extent, t.ncols + t.nrows);
  }
  if (chunks == 0)
    return CAFXG_OK;
  MLaunch L{};
  L.n = (uint32_t)tiles.size();
  L.total_chunks = chunks;
  L.max_iter = tiles[0].max_iter;
  L.out = out_base;
  L.sched = d->next_sched();
  L.zero = 0.0f;
  L.inline_coords = tiles[0].cx == nullptr;
  if (direct_counters) {
    // run_mandel_batch checked the same conditions and skips the reply copy
    if (tiles.size() > (size_t)kInlineTiles || !L.inline_coords)
      return fail(CAFXG_E_CONFIG, "internal: direct reply on an ineligible batch");
    L.direct = 1;
    L.tile_done = direct_counters;
  }
  MTile* dev_tiles = nullptr;
  if (tiles.size() <= (size_t)kInlineTiles) {
    for (size_t i = 0; i < tiles.size(); ++i)
      L.inl[i] = tiles[i];
  } else {
    size_t bytes = tiles.size() * sizeof(MTile);
    CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dev_tiles, bytes, stream));
    CAFXG_TRY(upload(d, dev_tiles, tiles.data(), bytes, stream));
    ctx->st_h2d += bytes;
    L.tiles = dev_tiles;
  }
  if (!skip_coords) {
    int e = mandel_coords_launch(L, precision, max_extent, stream);
    if (e != 0)
      return cuda_status((cudaError_t)e, "mandelbrot coordinate launch");
    ctx->st_launches++;
  }
  if (!coords_only) {
    bool safe = true;
    for (auto& t : tiles)
      safe = safe && deferred_safe(t);
    MandelLaunchCfg cfg = mandel_cfg(d, precision, L.max_iter, exact, safe, pixels);
    const auto l0 = std::chrono::steady_clock::now();
    int e = mandel_launch(L, precision, cfg, stream);
    ctx->st_phase_ns[5] += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                               std::chrono::steady_clock::now() - l0)
                               .count();
    if (e != 0)
      return cuda_status((cudaError_t)e, "mandelbrot launch");
    ctx->st_launches++;
  }
  if (dev_tiles)
    CAFXG_CUDA_TRY(cudaFreeAsync(dev_tiles, stream));
  return CAFXG_OK;
}

// Splits the request's tiles into row-band sub-tiles dealt cyclically to the
// devices (contiguous bands are load-imbalanced up to 1.15x).
static std::vector<std::vector<SubTile>> plan_mandel(
    const cafxg_mandel_desc* tiles, size_t n, size_t ndev) {
  std::vector<std::vector<SubTile>> per(ndev);
  uint64_t total = 0;
  for (size_t i = 0; i < n; ++i)
    total += (uint64_t)tiles[i].nrows * tiles[i].ncols;
  // band size: ~1M pixels when the request is large enough to share; a
  // single-device request of 1M..64M pixels goes in ~8 bands of >= 512K (four
  // for cfg1's 2M pixels), so copy-outs overlap the later bands' kernels
  // (a rank's 1/8 share of cfg3 is 32M pixels)
  static const uint64_t band_min = [] {  // CAFXG_BAND_MIN_KPX: experiments only
    const char* e = getenv("CAFXG_BAND_MIN_KPX");
    const int v = e ? atoi(e) : 0;
    return (v > 0 ? (uint64_t)v : 512ull) << 10;
  }();
  const uint64_t band_px = (ndev > 1 || total > (64ull << 20)) ? (1ull << 20)
                           : total >= (1ull << 20) ? std::max<uint64_t>((total + 7) / 8, band_min)
                                                   : UINT64_MAX;
  size_t next = 0;
  for (size_t i = 0; i < n; ++i) {
    const cafxg_mandel_desc& t = tiles[i];
    uint64_t px = (uint64_t)t.nrows * t.ncols;
    if (px == 0)
      continue;
    uint32_t rows_per = band_px == UINT64_MAX
                            ? t.nrows
                            : (uint32_t)std::max<uint64_t>(1, band_px / t.ncols);
    for (uint32_t r = 0; r < t.nrows; r += rows_per) {
      SubTile s;
      s.d = t;
      s.d.row0 = t.row0 + r;
      s.d.nrows = std::min(rows_per, t.nrows - r);
      s.d.out_offset = t.out_offset + (uint64_t)r * t.ncols;
      s.pixels = (uint64_t)s.d.nrows * s.d.ncols;
      per[next % ndev].push_back(s);
      ++next;
    }
  }
  return per;
}

static int stream_after(cudaStream_t b, cudaStream_t a);  // b waits for a's work so far
static int stream_after_pooled(Device* d, cudaStream_t b, cudaStream_t a);

// Submits one device's share: waves of sub-tiles, each a single launch into a
// device staging buffer followed by the copy-out on the d2h stream, so the
// PCIe transfer of wave w overlaps the compute of wave w+1.
static int submit_mandel_device(cafxg_ctx* ctx, Device* d,
                                const std::vector<SubTile>& subs,
                                uint32_t* host_out, bool out_pinned,
                                bool exact, Join* join) {
  cudaSetDevice(d->ordinal);
  std::lock_guard<std::mutex> g(d->submit_mu);
  static const uint64_t wave_px = [] {  // CAFXG_WAVE_MPX: experiments only
    const char* e = getenv("CAFXG_WAVE_MPX");
    const int v = e ? atoi(e) : 0;
    return (v > 0 ? (uint64_t)v : 32ull) << 20;
  }();
  uint32_t* staging = nullptr;  // pinned bounce buffer for pageable outputs
  uint64_t dev_px_total = 0;
  for (auto& s : subs)
    dev_px_total += s.pixels;
  if (!out_pinned) {
    staging = (uint32_t*)ctx->pinned.alloc(dev_px_total * 4);
    if (!staging)
      return fail(CAFXG_E_CONFIG, "mandelbrot: pinned staging allocation failed");
  }
  uint64_t staged = 0;
  std::vector<std::array<uint64_t, 3>> scat;  // (staging off, host off, px)
  size_t i = 0;
  // pixels still to schedule: waves shrink geometrically towards the end so
  // the copy-out left exposed after the last kernel is small
  uint64_t left = dev_px_total;
  // smallest wave: 2M pixels (launch overhead), 512K for small requests
  static const uint64_t big_min = [] {  // CAFXG_MIN_WAVE_MPX: experiments only
    const char* e = getenv("CAFXG_MIN_WAVE_MPX");
    const int v = e ? atoi(e) : 0;
    return (v > 0 ? (uint64_t)v : 2ull) << 20;
  }();
  static const uint64_t small_min = [] {  // CAFXG_SMALL_WAVE_KPX: experiments only
    const char* e = getenv("CAFXG_SMALL_WAVE_KPX");
    const int v = e ? atoi(e) : 0;
    return (v > 0 ? (uint64_t)v : 512ull) << 10;
  }();
  const uint64_t min_wave = dev_px_total >= (64ull << 20) ? big_min : small_min;
  // Small, shallow requests (<= 4M pixels, max_iter <= 256: cfg1) are bound by
  // the copy-out, not the kernel: one small first wave starts the copy engine
  // early and everything else goes in a second wave whose contiguous bands
  // leave in one copy (2 MB copies ran at ~45 GB/s, the link does ~55).
  // CAFXG_SMALL_PLAN=0: the geometric waves everywhere (experiments).
  static const bool small_plan_on = [] {
    const char* e = getenv("CAFXG_SMALL_PLAN");
    return !(e && e[0] == '0');
  }();
  uint32_t req_maxit = 0;
  for (auto& sb : subs)
    req_maxit = std::max(req_maxit, sb.d.max_iter);
  const bool two_waves = small_plan_on && dev_px_total <= (4ull << 20) && req_maxit <= 256;
  // CAFXG_TRACE=1: per-wave device timeline on stderr (debug aid)
  static const bool trace = [] {
    const char* e = getenv("CAFXG_TRACE");
    return e && e[0] == '1';
  }();
  std::vector<std::array<cudaEvent_t, 3>> tev;
  std::vector<double> thost;  // host clock at each wave's start / after its launches
  const double t_entry = trace_now_ms();
  // waves alternate between the two compute streams (both ordered after the
  // device's earlier work; compute is ordered after both at the end)
  CAFXG_TRY(stream_after(d->compute2, d->compute));
  uint32_t wave = 0;
  while (i < subs.size()) {
    // (the two-wave plan keeps one stream: the first wave then runs alone and
    // its copy starts sooner)
    cudaStream_t ks = ((wave++ & 1) && !two_waves) ? d->compute2 : d->compute;
    // group a wave (same precision)
    size_t j = i;
    uint64_t px = 0;
    int prec = subs[i].d.precision;
    const uint64_t cap =
        two_waves ? (wave == 1 ? min_wave : UINT64_MAX)
                  : std::max<uint64_t>(std::min<uint64_t>(wave_px, left / 4), min_wave);
    while (j < subs.size() && subs[j].d.precision == prec &&
           (px == 0 || px + subs[j].pixels <= cap)) {
      px += subs[j].pixels;
      ++j;
    }
    uint32_t* dout = nullptr;
    CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dout, px * 4, ks));
    std::vector<MTile> mt(j - i);
    uint32_t chunks = 0, maxit = 0;
    uint64_t off = 0;
    for (size_t k = i; k < j; ++k) {
      fill_mtile(mt[k - i], subs[k].d, off, chunks);
      chunks += tile_chunks(subs[k].d.nrows, subs[k].d.ncols, subs[k].d.precision);
      maxit = std::max(maxit, subs[k].d.max_iter);
      off += subs[k].pixels;
    }
    if (trace) {
      tev.push_back({});
      for (auto& e : tev.back())
        cudaEventCreate(&e);
      cudaEventRecord(tev.back()[0], ks);
      thost.push_back(trace_now_ms());
    }
    CAFXG_TRY(launch_mandel(ctx, d, dout, mt, chunks, prec, maxit, exact, px, ks));
    if (trace)
      thost.push_back(trace_now_ms());
    if (trace)
      cudaEventRecord(tev.back()[1], ks);
    CAFXG_TRY(stream_after_pooled(d, d->d2h, ks));
    off = 0;
    // copies of consecutive sub-tiles that are contiguous on both sides
    // (row bands of one tile into a pinned image; any run into the staging
    // buffer) go out as one cudaMemcpyAsync
    uint32_t* run_dst = nullptr;
    uint64_t run_src = 0, run_px = 0;
    auto flush_run = [&]() -> int {
      if (run_px) {
        CAFXG_CUDA_TRY(cudaMemcpyAsync(run_dst, dout + run_src, run_px * 4,
                                       cudaMemcpyDeviceToHost, d->d2h));
        ctx->st_d2h += run_px * 4;
      }
      run_px = 0;
      return CAFXG_OK;
    };
    for (size_t k = i; k < j; ++k) {
      uint32_t* dst;
      if (out_pinned) {
        dst = host_out + subs[k].d.out_offset;
      } else {
        dst = staging + staged;
        scat.push_back({staged, subs[k].d.out_offset, subs[k].pixels});
        staged += subs[k].pixels;
      }
      if (run_px && dst != run_dst + run_px)
        CAFXG_TRY(flush_run());
      if (!run_px) {
        run_dst = dst;
        run_src = off;
      }
      run_px += subs[k].pixels;
      off += subs[k].pixels;
    }
    CAFXG_TRY(flush_run());
    CAFXG_CUDA_TRY(cudaFreeAsync(dout, d->d2h));
    if (trace)
      cudaEventRecord(tev.back()[2], d->d2h);
    left -= px;
    i = j;
  }
  CAFXG_TRY(stream_after(d->compute, d->compute2));
  if (trace && !tev.empty()) {
    cudaError_t se = cudaEventSynchronize(tev.back()[2]);
    for (size_t w = 0; w < tev.size(); ++w) {
      float a = -1, b = -1, c = -1;
      cudaError_t e1 = cudaEventElapsedTime(&a, tev[0][0], tev[w][0]);
      cudaError_t e2 = cudaEventElapsedTime(&b, tev[0][0], tev[w][1]);
      cudaError_t e3 = cudaEventElapsedTime(&c, tev[0][0], tev[w][2]);
      if (se || e1 || e2 || e3)
        fprintf(stderr, "cafxg trace errors %d %d %d %d\n", (int)se, (int)e1, (int)e2, (int)e3);
      fprintf(stderr, "cafxg trace wave %zu: kernel %.3f..%.3f ms, copy done %.3f ms\n", w, a, b,
              c);
    }
    for (size_t w = 0; w + 1 < thost.size(); w += 2)
      fprintf(stderr, "cafxg trace host: wave %zu issued %.3f..%.3f ms after entry\n", w / 2,
              thost[w] - t_entry, thost[w + 1] - t_entry);
    for (auto& w : tev)
      for (auto& e : w)
        cudaEventDestroy(e);
    cudaGetLastError();
  }
  return push_completion(ctx, d, d->d2h,
                         [ctx, staging, scat = std::move(scat), host_out, join](int st) {
                           if (staging) {
                             if (st == CAFXG_OK)
                               for (auto& s : scat)
                                 std::memcpy(host_out + s[1], staging + s[0], s[2] * 4);
                             ctx->pinned.free(staging);
                           }
                           join->part_done(st);
                         });
}

static int mandel_submit_impl(cafxg_ctx* ctx, const cafxg_mandel_desc* tiles,
                              size_t n, uint32_t* host_out, cafxg_done_fn done,
                              void* user) {
  if (!ctx || (n && !tiles) || (n && !host_out))
    return fail(CAFXG_E_CONFIG, "mandelbrot_submit: null argument");
  uint64_t out_elems = 0;
  bool exact = false;
  for (size_t i = 0; i < n; ++i) {
    CAFXG_TRY(validate_mandel(tiles[i]));
    out_elems = std::max<uint64_t>(
        out_elems, tiles[i].out_offset + (uint64_t)tiles[i].nrows * tiles[i].ncols);
    exact = exact || use_exact(ctx, tiles[i]);
  }
  bool pinned = host_is_pinned(host_out, out_elems * 4);
  auto plan = plan_mandel(tiles, n, ctx->devs.size());
  Join* join = new Join;
  join->done = done;
  join->user = user;
  int parts = 0;
  for (auto& p : plan)
    parts += !p.empty();
  if (parts == 0) {
    // nothing to compute: complete through device 0's completion thread so
    // the callback still runs off the caller's thread
    join->remaining = 1;
    Device* d = ctx->devs[0].get();
    cudaSetDevice(d->ordinal);
    std::lock_guard<std::mutex> g(d->submit_mu);
    return push_completion(ctx, d, d->compute, [join](int st) { join->part_done(st); });
  }
  join->remaining = parts;
  ctx->st_requests++;
  for (size_t k = 0; k < plan.size(); ++k) {
    if (plan[k].empty())
      continue;
    int s = submit_mandel_device(ctx, ctx->devs[k].get(), plan[k], host_out,
                                 pinned, exact, join);
    if (s != CAFXG_OK) {
      // parts already submitted still report through the join
      std::string err = t_last_error;
      join->part_done(s);
      for (size_t r = k + 1; r < plan.size(); ++r)
        if (!plan[r].empty())
          join->part_done(s);
      t_last_error = err;
      return CAFXG_OK;  // the error is delivered through `done`
    }
  }
  return CAFXG_OK;
}

// ---- sgemm ---------------------------------------------------------------------------

static int validate_sgemm(cafxg_sgemm_desc& d) {
  if (d.lda == 0) d.lda = d.K;
  if (d.ldb == 0) d.ldb = d.N;
  if (d.ldc == 0) d.ldc = d.N;
  if (d.lda < d.K || d.ldb < d.N || d.ldc < d.N)
    return fail(CAFXG_E_OUT_OF_RANGE, "sgemm: leading dimension below extent");
  if (d.mode > CAFXG_SGEMM_3XTF32)
    return fail(CAFXG_E_CONFIG, "sgemm: bad mode");
  if (d.M > (1u << 30) || d.N > (1u << 30) || d.K > (1u << 30))
    return fail(CAFXG_E_OUT_OF_RANGE, "sgemm: dimension too large");
  return CAFXG_OK;
}

// Runs C = A*B on one device with device pointers.
static int sgemm_on_device(cafxg_ctx* ctx, Device* d, const cafxg_sgemm_desc& g,
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
  bool supported = sgemm_tc_supported(g.M, g.N, g.K, g.lda, g.ldb, g.ldc);
  bool tc = supported && (g.mode == CAFXG_SGEMM_3XTF32 || (g.mode == CAFXG_SGEMM_AUTO && auto_tc));
  if (g.mode == CAFXG_SGEMM_3XTF32 && !tc)
    return fail(CAFXG_E_CONFIG,
                "sgemm: shape not supported by the 3xTF32 kernel (see cafxg.h)");
  if (tc) {
    size_t sb = sgemm_tc_scratch_bytes(g.M, g.N, g.K);
    void* scratch = nullptr;
    CAFXG_CUDA_TRY(cudaMallocAsync(&scratch, sb, stream));
    int launches = 0;
    int e = sgemm_tc_launch(A, B, C, g.M, g.N, g.K, g.lda, g.ldb, g.ldc, scratch,
                            d->sms, stream, &launches);
    ctx->st_launches += launches;
    CAFXG_CUDA_TRY(cudaFreeAsync(scratch, stream));
    if (e != 0)
      return cuda_status((cudaError_t)e, "sgemm 3xtf32 launch");
    return CAFXG_OK;
  }
  int e = sgemm_simt_launch(A, B, C, g.M, g.N, g.K, g.lda, g.ldb, g.ldc, stream);
  if (e != 0)
    return cuda_status((cudaError_t)e, "sgemm simt launch");
  ctx->st_launches++;
  return CAFXG_OK;
}

static int ensure_nccl(cafxg_ctx* ctx) {
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


static bool trace_on() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}

static int stream_after(cudaStream_t b, cudaStream_t a) {
  cudaEvent_t ev;
  CAFXG_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CAFXG_CUDA_TRY(cudaEventRecord(ev, a));
  CAFXG_CUDA_TRY(cudaStreamWaitEvent(b, ev, 0));
  cudaEventDestroy(ev);  // released once it completes
  return CAFXG_OK;
}

// The same with the device's reusable ordering event (caller holds
// d->submit_mu): the wait captures the record, so the event is free again at
// once.
static int stream_after_pooled(Device* d, cudaStream_t b, cudaStream_t a) {
  if (!d->order_ev)
    CAFXG_CUDA_TRY(cudaEventCreateWithFlags(&d->order_ev, cudaEventDisableTiming));
  CAFXG_CUDA_TRY(cudaEventRecord(d->order_ev, a));
  CAFXG_CUDA_TRY(cudaStreamWaitEvent(b, d->order_ev, 0));
  return CAFXG_OK;
}

static cudaEvent_t pooled_event(Device* d) {
  if (!d->ev_pool.empty()) {
    cudaEvent_t e = d->ev_pool.back();
    d->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return e;
}

// Host-request pipeline for one device's C rows [r0, r1) with B already in
// device memory (dB, K x N): B is split once (tf32 hi/lo, transposed), then
// per block of R rows: H2D of A_i on the upload stream -> hi/lo split + 3xTF32
// GEMM on the compute stream -> D2H of C_i on the download stream. A and C
// blocks are double-buffered, so PCIe traffic in both directions overlaps the
// tensor-core work. Completion is recorded on d2h.
static bool sgemm_pipeline_eligible(const cafxg_sgemm_desc& g, uint32_t rows) {
  return g.mode != CAFXG_SGEMM_FFMA && rows >= 1024 && rows % 128 == 0 &&
         sgemm_tc_supported(128, g.N, g.K, g.K, g.N, g.N);
}

// hostB: when non-null, B (K x N, host) is uploaded here on the upload
// stream, ahead of the A blocks, instead of by the caller into dB: the first A
// block then follows B over PCIe without waiting for B's split.
static int sgemm_pipeline_device(cafxg_ctx* ctx, Device* d, const cafxg_sgemm_desc& g,
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
  float *Bh = nullptr, *Bl = nullptr, *Ah = nullptr, *Al = nullptr;
  float* dA[2] = {nullptr, nullptr};
  float* dC[2] = {nullptr, nullptr};
  cudaStream_t cs = d->compute;
  // buffers carved from the device's grow-only workspace (a stream-ordered
  // allocation and free per buffer and request cost more host time than the
  // GEMMs of a 1024^3 request); 256-byte aligned pieces
  {
    const size_t pieces[8] = {N * K, N * K, (size_t)R * K, (size_t)R * K, (size_t)R * K,
                              (size_t)R * K, (size_t)R * N, (size_t)R * N};
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
    float** dst[8] = {&Bh, &Bl, &Ah, &Al, &dA[0], &dA[1], &dC[0], &dC[1]};
    uint8_t* base = reinterpret_cast<uint8_t*>(d->sgemm_ws);
    for (int i = 0; i < 8; ++i) {
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
  int e = sgemm_tc_split_b(dB, (int)N, (int)K, (int)N, Bh, Bl, cs);
  if (e != 0)
    return cuda_status((cudaError_t)e, "sgemm: B split");
  ctx->st_launches++;
  // tensor maps encoded once per request: every block reuses Ah/Al (R rows)
  // and Bh/Bl
  SgemmTcMaps maps;
  if (int me = sgemm_tc_make_maps(Ah, Al, (int)R, Bh, Bl, (int)N, (int)K, &maps))
    return cuda_status((cudaError_t)me, "sgemm: tensor maps");
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
    // upload A block (slot free once block i-2's split consumed it)
    if (i >= 2)
      cudaStreamWaitEvent(d->h2d, ev_split[i - 2], 0);
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
    e = sgemm_tc_split_a(dA[slot], (int)K, (int)m, (int)K, Ah, Al, cs);
    cudaEventRecord(mk(ev_split), cs);
    if (e == 0)
      e = sgemm_tc_gemm_maps(&maps, dC[slot], (int)m, (int)N, (int)K, (int)N, cs,
                             sgemm_tc_splits((int)m, (int)N, (int)K, d->sms));
    if (e != 0)
      status = cuda_status((cudaError_t)e, "sgemm: 3xtf32 launch");
    ctx->st_launches += 2;
    tmark("gemm", cs);
    cudaEventRecord(mk(ev_gemm), cs);
    cudaStreamWaitEvent(d->d2h, ev_gemm.back(), 0);
    if (status == CAFXG_OK)
      status = cuda_status(cudaMemcpy2DAsync(C + (size_t)(r0 + b0) * g.ldc, (size_t)g.ldc * 4,
                                             dC[slot], N * 4, N * 4, m,
                                             cudaMemcpyDeviceToHost, d->d2h),
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
static bool sgemm_tiled2d_eligible(const cafxg_sgemm_desc& g) {
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

static int sgemm_tiled2d_device(cafxg_ctx* ctx, Device* d, const cafxg_sgemm_desc& g,
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
  if (int me = sgemm_tc_make_maps(Ah, Al, (int)M, Bh, Bl, (int)N, (int)K, &maps))
    return cuda_status((cudaError_t)me, "sgemm: tensor maps");
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
    int e = sgemm_tc_gemm_maps(&maps, cblk, (int)mi, (int)nj, (int)K, (int)N, cs,
                               sgemm_tc_splits((int)mi, (int)nj, (int)K, d->sms), (int)m0,
                               (int)n0);
    ctx->st_launches++;
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
static int sgemm_submit_impl(cafxg_ctx* ctx, const cafxg_sgemm_desc* desc,
                             const float* A, const float* B, float* C,
                             cafxg_done_fn done, void* user) {
  if (!ctx || !desc)
    return fail(CAFXG_E_CONFIG, "sgemm_submit: null argument");
  cafxg_sgemm_desc g = *desc;
  CAFXG_TRY(validate_sgemm(g));
  if ((g.M && g.K && !A) || (g.K && g.N && !B) || (g.M && g.N && !C))
    return fail(CAFXG_E_CONFIG, "sgemm_submit: null matrix");
  size_t G = ctx->devs.size();
  // devices used: only split when every block gets rows and K divides evenly
  size_t use = 1;
  bool nccl = false;
  if (G > 1 && g.M >= G * 128 && g.K % G == 0 && g.ldb == g.N) {
    use = G;
    // NCCL all-gather over NVLink; without it (virtual devices, or NCCL not
    // loadable) the slices are replicated by peer copies on the copy engines
    nccl = ensure_nccl(ctx) == CAFXG_OK;
    clear_last_error();
  }
  Join* join = new Join;
  join->done = done;
  join->user = user;
  join->remaining = (int)use;
  ctx->st_requests++;
  if (use == 1 && sgemm_tiled2d_eligible(g)) {
    Device* d = ctx->devs[0].get();
    std::lock_guard<std::mutex> lk(d->submit_mu);
    cudaSetDevice(d->ordinal);
    int s = sgemm_tiled2d_device(ctx, d, g, A, B, C);
    if (s != CAFXG_OK) {
      // queued work may still read the host buffers: report after it
      push_completion(ctx, d, d->d2h, [join, s](int) { join->part_done(s); });
      return CAFXG_OK;
    }
    if (push_completion(ctx, d, d->d2h, [join](int st) { join->part_done(st); }) != CAFXG_OK)
      join->part_done(CAFXG_E_DOWN);
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
  const bool defer_b = use == 1 && g.M && g.ldb == g.N && sgemm_pipeline_eligible(g, g.M);
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
  if (status == CAFXG_OK && use > 1 && nccl) {
    ctx->nccl.GroupStart();
    for (size_t k = 0; k < use; ++k) {
      size_t cnt = (size_t)g.K / use * g.ldb;
      ctx->nccl.AllGather(dB[k] + cnt * k, dB[k], cnt, ncclFloat32, ctx->comms[k],
                          ctx->devs[k]->compute);
    }
    if (ctx->nccl.GroupEnd() != ncclSuccess)
      status = fail(CAFXG_E_DOWN, "sgemm: NCCL all-gather of B failed");
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
      else if (push_completion(ctx, d, d->d2h, [join](int st) { join->part_done(st); }) !=
               CAFXG_OK)
        join->part_done(CAFXG_E_DOWN);
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
    if (s != CAFXG_OK) {
      // still route the failure through the completion thread
      push_completion(ctx, d, d->compute, [join, s](int) { join->part_done(s); });
    } else {
      int ps = push_completion(ctx, d, d->compute, [join](int st) { join->part_done(st); });
      if (ps != CAFXG_OK)
        join->part_done(ps);
    }
  }
  return CAFXG_OK;
}

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
};

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

static void actor_unref(cafxg_actor* a) {
  if (a->refs.fetch_sub(1) == 1)
    delete a;
}

// Completes one actor request: the caller's callback, then the bookkeeping.
// `account` = false when the caller settles the context counters for a whole
// batch at once (st_requests / actor_open / the sync notification).
static void finish_request(Request* r, int status, bool account = true) {
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
static void finish_batch(cafxg_ctx* ctx, std::vector<Request*> batch, uint32_t* bounce,
                         int status);

// Callback thread: runs reply jobs (slices of large batches, copy pieces).
static void callback_loop(cafxg_ctx* ctx) {
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
    job();
  }
}

static void finish_batch(cafxg_ctx* ctx, std::vector<Request*> batch, uint32_t* bounce,
                         int status) {
  constexpr size_t kSlice = 1024;
  const size_t n = batch.size();
  // src: the staging buffer to copy replies out of (nullptr: already placed)
  auto run_slice = [ctx, status](Request* const* rs, size_t cnt, uint64_t pix_off,
                                 const uint32_t* src) {
    uint64_t o = pix_off;
    for (size_t i = 0; i < cnt; ++i) {
      Request* r = rs[i];
      if (src && status == CAFXG_OK)
        std::memcpy(r->out, src + o, r->pixels * 4);
      o += r->pixels;
      finish_request(r, status, false);
    }
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

static inline uint64_t now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// One batch of Mandelbrot requests (same precision) on one device: one launch
// over every tile of every request into a device staging slot; small batches
// into pinned replies are then copied out by that kernel itself (direct
// reply), others by one scatter launch straight into the pinned reply buffers
// (or one D2H into a pinned bounce buffer + host memcpy for pageable replies).
static void run_mandel_batch(cafxg_ctx* ctx, Device* d, std::vector<Request*> batch) {
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
      direct = tp % 4 == 0 && tp <= kDirectTilePx;
    }
  }
  if (!d->stage[0]) {
    // first batch on this device: the whole ring at the batch cap, so later
    // batches never allocate (one request above the cap still grows its slot)
    for (int i = 0; i < kMaxInflight; ++i) {
      const size_t cap = kMaxBatchPx * 4 + kStageTail;
      if (cudaMalloc((void**)&d->stage[i], cap) == cudaSuccess &&
          cudaMemset(d->stage[i] + cap - kStageTail, 0, kStageTail) == cudaSuccess) {
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
          cudaMemset(d->stage[slot] + cap - kStageTail, 0, kStageTail) != cudaSuccess) {
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
  status = launch_mandel(ctx, d, dout, mt, chunks, prec, maxit, exact, px, ks, counters);
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

static Device* pick_device(cafxg_ctx* ctx) {
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

static void dispatcher_loop(cafxg_ctx* ctx) {
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
      if (!r->actor->alive.load()) {
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
        g.mode = CAFXG_SGEMM_AUTO;
        int s = sgemm_submit_impl(
            ctx, &g, r->a, r->b, (float*)r->out,
            [](void* u, int st) { finish_request((Request*)u, st); }, r);
        if (s != CAFXG_OK)
          push_completion(ctx, d, d->compute, [r, s](int) { finish_request(r, s); });
        ctx->st_requests--;  // counted by finish_request
        break;
      }
      if (!batch.empty() &&
          (r->precision != batch[0]->precision ||
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
      run_mandel_batch(ctx, d, std::move(batch));
      ctx->st_batch_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                              std::chrono::steady_clock::now() - b0)
                              .count();
    }
  }
}

static void wake_dispatcher(cafxg_ctx* ctx) {
  {
    std::lock_guard<std::mutex> lk(ctx->disp_mu);
    ctx->disp_wake = true;
  }
  ctx->disp_cv.notify_one();
}

}  // namespace cafxg

// =====================================================================================
// C ABI
// =====================================================================================

// No C++ exception crosses the ABI: functions that allocate on the host are
// function-try-blocks that turn std::bad_alloc and friends into an error
// status (config_error) with the message in cafxg_last_error().
extern "C" {

int cafxg_abi_version(void) { return CAFXG_ABI_VERSION; }

const char* cafxg_status_string(int s) {
  switch (s) {
    case CAFXG_OK: return "none";
    case CAFXG_E_UNKNOWN_TYPE: return "unknown_type";
    case CAFXG_E_OUT_OF_RANGE: return "out_of_range";
    case CAFXG_E_TYPE_MISMATCH: return "type_mismatch";
    case CAFXG_E_INTERFACE_MISMATCH: return "interface_mismatch";
    case CAFXG_E_CONFIG: return "config_error";
    case CAFXG_E_SPAWN: return "spawn_error";
    case CAFXG_E_TIMEOUT: return "request_timeout";
    case CAFXG_E_DOWN: return "request_down";
    default: return "unknown";
  }
}

const char* cafxg_last_error(void) { return t_last_error.c_str(); }

int cafxg_open(uint64_t device_mask, cafxg_ctx** out) {
  if (!out)
    return fail(CAFXG_E_CONFIG, "open: null out");
  *out = nullptr;
  try {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      return fail(CAFXG_E_SPAWN, "no CUDA device visible (%s)",
                  e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
    }
    auto ctx = std::make_unique<cafxg_ctx>();
    std::vector<int> ords;
    for (int i = 0; i < n && i < 64; ++i)
      if (!device_mask || (device_mask >> i & 1))
        ords.push_back(i);
    const char* vd = getenv("CAFXG_VIRTUAL_DEVICES");
    int vcount = vd ? atoi(vd) : 0;
    if (vcount > 1 && ords.size() == 1) {
      ords.assign(std::min(vcount, 64), ords[0]);
      ctx->virtual_devs = true;
    }
    for (int i : ords) {
      auto d = std::make_unique<Device>();
      d->ordinal = i;
      CAFXG_CUDA_TRY(cudaSetDevice(i));
      cudaDeviceProp prop{};
      CAFXG_CUDA_TRY(cudaGetDeviceProperties(&prop, i));
      if (prop.major != 10)
        return fail(CAFXG_E_SPAWN, "device %d is sm_%d%d; libcafxg is built for sm_100a",
                    i, prop.major, prop.minor);
      d->sms = prop.multiProcessorCount;
      CAFXG_CUDA_TRY(cudaStreamCreateWithFlags(&d->compute, cudaStreamNonBlocking));
      CAFXG_CUDA_TRY(cudaStreamCreateWithFlags(&d->compute2, cudaStreamNonBlocking));
      CAFXG_CUDA_TRY(cudaStreamCreateWithFlags(&d->d2h, cudaStreamNonBlocking));
      CAFXG_CUDA_TRY(cudaStreamCreateWithFlags(&d->h2d, cudaStreamNonBlocking));
      CAFXG_CUDA_TRY(cudaMalloc(&d->sched, kSchedSlots * 2 * sizeof(uint32_t)));
      CAFXG_CUDA_TRY(cudaMemset(d->sched, 0, kSchedSlots * 2 * sizeof(uint32_t)));
      CAFXG_CUDA_TRY(cudaHostAlloc((void**)&d->up_base, kUpSlots * kUpSlotBytes,
                                   cudaHostAllocPortable));
      for (auto& ev : d->up_ev)
        CAFXG_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      cudaMemPool_t pool;
      CAFXG_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, i));
      uint64_t thr = UINT64_MAX;
      CAFXG_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
      ctx->devs.push_back(std::move(d));
    }
    if (ctx->devs.empty())
      return fail(CAFXG_E_SPAWN, "device_mask selects no visible device");
    const char* ex = getenv("CAFXG_EXACT_STEP");
    ctx->force_exact = ex && ex[0] == '1';
    cafxg_ctx* c = ctx.release();
    for (auto& d : c->devs)
      d->completer = std::thread(completion_loop, c, d.get());
    c->dispatcher = std::thread(dispatcher_loop, c);
    unsigned hw = std::thread::hardware_concurrency();
    unsigned ncb = std::max(1u, std::min(8u, hw / 4));
    for (unsigned i = 0; i < ncb; ++i)
      c->cb_threads.emplace_back(callback_loop, c);
    *out = c;
    return CAFXG_OK;
  } catch (const std::exception& ex) {
    return fail(CAFXG_E_SPAWN, "open: %s", ex.what());
  }
}

int cafxg_sync(cafxg_ctx* ctx) {
  if (!ctx)
    return fail(CAFXG_E_CONFIG, "sync: null ctx");
  std::unique_lock<std::mutex> lk(ctx->sync_mu);
  while (!(ctx->completed == ctx->submitted && ctx->actor_open.load() == 0))
    ctx->sync_cv.wait_for(lk, std::chrono::milliseconds(1));
  return CAFXG_OK;
}

int cafxg_close(cafxg_ctx* ctx) try {
  if (!ctx)
    return CAFXG_OK;
  if ((trace_on() || getenv("CAFXG_STATS")) && ctx->st_batches.load())
    fprintf(stderr, "cafxg: %llu batches, dispatcher submit time %.3f ms (%.2f us/batch)\n",
            (unsigned long long)ctx->st_batches.load(), ctx->st_batch_ns.load() / 1e6,
            ctx->st_batch_ns.load() / 1e3 / ctx->st_batches.load());
  if ((trace_on() || getenv("CAFXG_STATS")) && ctx->st_batches.load())
    fprintf(stderr, "cafxg:   %llu batches replied by the escape kernel (direct)\n",
            (unsigned long long)ctx->st_direct.load());
  if ((trace_on() || getenv("CAFXG_STATS")) && ctx->st_batches.load()) {
    const char* nm[6] = {"build", "kernel launch", "copy-stream order", "reply launch",
                         "record+completion", "(of which the escape-kernel launch call)"};
    for (int i = 0; i < 6; ++i)
      fprintf(stderr, "cafxg:   %s %.2f us/batch\n", nm[i],
              ctx->st_phase_ns[i].load() / 1e3 / ctx->st_batches.load());
  }
  {
    std::lock_guard<std::mutex> lk(ctx->disp_mu);
    ctx->disp_stop = true;
  }
  ctx->disp_cv.notify_all();
  if (ctx->dispatcher.joinable())
    ctx->dispatcher.join();
  // completion threads may still hand slices to the callback threads, so
  // those stop last (after the completion threads below)
  for (auto& d : ctx->devs) {
    {
      std::lock_guard<std::mutex> lk(d->cq_mu);
      d->stop = true;
    }
    d->cq_cv.notify_all();
    if (d->completer.joinable())
      d->completer.join();
  }
  {
    std::lock_guard<std::mutex> lk(ctx->cb_mu);
    ctx->cb_stop = true;
  }
  ctx->cb_cv.notify_all();
  for (auto& t : ctx->cb_threads)
    if (t.joinable())
      t.join();
  for (auto& d : ctx->devs) {
    cudaSetDevice(d->ordinal);
    cudaStreamSynchronize(d->compute);
    cudaStreamSynchronize(d->d2h);
    for (auto ev : d->ev_free)
      cudaEventDestroy(ev);
    for (auto ev : d->up_ev)
      cudaEventDestroy(ev);
    for (auto ev : d->ev_pool)
      cudaEventDestroy(ev);
    if (d->sgemm_ws)
      cudaFree(d->sgemm_ws);
    if (d->order_ev)
      cudaEventDestroy(d->order_ev);
    cudaFreeHost(d->up_base);
    for (int i = 0; i < kMaxInflight; ++i) {
      if (d->stage[i])
        cudaFree(d->stage[i]);
      if (d->stage_ev[i])
        cudaEventDestroy(d->stage_ev[i]);
    }
    cudaFree(d->sched);
    cudaStreamSynchronize(d->h2d);
    cudaStreamSynchronize(d->compute2);
    cudaStreamDestroy(d->compute2);
    cudaStreamDestroy(d->compute);
    cudaStreamDestroy(d->d2h);
    cudaStreamDestroy(d->h2d);
  }
  if (!ctx->comms.empty())
    for (auto c : ctx->comms)
      ctx->nccl.CommDestroy(c);
  delete ctx;
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_close: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_close: unknown exception");
}

int cafxg_device_count(const cafxg_ctx* ctx) { return ctx ? (int)ctx->devs.size() : 0; }

int cafxg_host_alloc(cafxg_ctx* ctx, size_t bytes, void** ptr) try {
  if (!ctx || !ptr)
    return fail(CAFXG_E_CONFIG, "host_alloc: null argument");
  *ptr = ctx->pinned.alloc(bytes ? bytes : 1);
  if (!*ptr)
    return fail(CAFXG_E_OUT_OF_RANGE, "host_alloc: cudaHostAlloc of %zu bytes failed", bytes);
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_host_alloc: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_host_alloc: unknown exception");
}

int cafxg_host_free(cafxg_ctx* ctx, void* ptr) {
  if (!ctx)
    return fail(CAFXG_E_CONFIG, "host_free: null ctx");
  if (!ptr)
    return CAFXG_OK;
  return ctx->pinned.free(ptr) ? CAFXG_OK
                               : fail(CAFXG_E_CONFIG, "host_free: pointer not from host_alloc");
}

int cafxg_host_register(cafxg_ctx* ctx, void* ptr, size_t bytes) try {
  if (!ctx || !ptr || !bytes)
    return fail(CAFXG_E_CONFIG, "host_register: bad argument");
  CAFXG_CUDA_TRY(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_host_register: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_host_register: unknown exception");
}

int cafxg_host_unregister(cafxg_ctx* ctx, void* ptr) {
  if (!ctx || !ptr)
    return fail(CAFXG_E_CONFIG, "host_unregister: bad argument");
  CAFXG_CUDA_TRY(cudaHostUnregister(ptr));
  return CAFXG_OK;
}

int cafxg_mandelbrot_submit(cafxg_ctx* ctx, const cafxg_mandel_desc* tiles, size_t n,
                            uint32_t* host_out, cafxg_done_fn done, void* user) {
  try {
    return mandel_submit_impl(ctx, tiles, n, host_out, done, user);
  } catch (const std::exception& ex) {
    return fail(CAFXG_E_CONFIG, "mandelbrot_submit: %s", ex.what());
  }
}

namespace {
struct Waiter {
  std::mutex mu;
  std::condition_variable cv;
  bool fired = false;
  int status = CAFXG_OK;
  std::string err;
  static void cb(void* u, int s) {
    auto* w = static_cast<Waiter*>(u);
    std::lock_guard<std::mutex> g(w->mu);
    w->fired = true;
    w->status = s;
    if (s != CAFXG_OK)
      w->err = t_last_error;
    w->cv.notify_all();
  }
  int wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return fired; });
    if (status != CAFXG_OK)
      set_last_error("%s", err.c_str());
    return status;
  }
};
}  // namespace

int cafxg_mandelbrot(cafxg_ctx* ctx, const cafxg_mandel_desc* tiles, size_t n,
                     uint32_t* host_out) try {
  Waiter w;
  int s = cafxg_mandelbrot_submit(ctx, tiles, n, host_out, &Waiter::cb, &w);
  if (s != CAFXG_OK)
    return s;
  return w.wait();
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_mandelbrot: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_mandelbrot: unknown exception");
}

int cafxg_mandelbrot_device(cafxg_ctx* ctx, int device, const cafxg_mandel_desc* tiles,
                            size_t n, uint32_t* dev_out, void* stream) {
  if (!ctx || device < 0 || device >= (int)ctx->devs.size() || (n && (!tiles || !dev_out)))
    return fail(CAFXG_E_CONFIG, "mandelbrot_device: bad argument");
  try {
    Device* d = ctx->devs[device].get();
    bool exact = false;
    std::vector<MTile> mt;
    mt.reserve(n);
    uint32_t chunks = 0, maxit = 0;
    uint64_t px = 0, lo = UINT64_MAX, hi = 0;
    int prec = n ? (int)tiles[0].precision : 0;
    for (size_t i = 0; i < n; ++i) {
      CAFXG_TRY(validate_mandel(tiles[i]));
      if ((int)tiles[i].precision != prec)
        return fail(CAFXG_E_CONFIG, "mandelbrot_device: mixed precisions in one launch");
      uint64_t tp = (uint64_t)tiles[i].nrows * tiles[i].ncols;
      if (tp == 0)
        continue;  // empty tiles own no chunks
      lo = std::min<uint64_t>(lo, tiles[i].out_offset);
      hi = std::max<uint64_t>(hi, tiles[i].out_offset + tp);
    }
    if (hi > lo && hi - lo >= (1ull << 32))
      return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot_device: one launch spans >= 2^32 counts");
    for (size_t i = 0; i < n; ++i) {
      uint64_t tp = (uint64_t)tiles[i].nrows * tiles[i].ncols;
      if (tp == 0)
        continue;
      exact = exact || use_exact(ctx, tiles[i]);
      MTile m;
      fill_mtile(m, tiles[i], tiles[i].out_offset - lo, chunks);
      mt.push_back(m);
      chunks += tile_chunks(tiles[i].nrows, tiles[i].ncols, tiles[i].precision);
      maxit = std::max(maxit, tiles[i].max_iter);
      px += tp;
    }
    if (mt.empty())
      return CAFXG_OK;
    cudaSetDevice(d->ordinal);
    cudaStream_t s = stream ? (cudaStream_t)stream : d->compute;
    return launch_mandel(ctx, d, dev_out + lo, mt, chunks, prec, maxit, exact, px, s);
  } catch (const std::exception& ex) {
    return fail(CAFXG_E_CONFIG, "mandelbrot_device: %s", ex.what());
  }
}

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
  Device* d = ctx->devs[device].get();
  cudaSetDevice(d->ordinal);
  return sgemm_on_device(ctx, d, g, A, B, C, stream ? (cudaStream_t)stream : d->compute);
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_sgemm_device: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_sgemm_device: unknown exception");
}

// ---- actors --------------------------------------------------------------------

int cafxg_spawn(cafxg_ctx* ctx, const char* kernel_name, const uint64_t* dims, size_t ndims,
                cafxg_actor** out) try {
  if (!ctx || !kernel_name || !out)
    return fail(CAFXG_E_CONFIG, "spawn: null argument");
  *out = nullptr;
  Kernel k;
  if (!std::strcmp(kernel_name, "mandelbrot")) {
    k = Kernel::mandelbrot;
  } else if (!std::strcmp(kernel_name, "matrix_multiply")) {
    k = Kernel::matrix_multiply;
    // spawn_cl<float*(float*,float*)>(src, "matrix_multiply", {size, size})
    if (ndims != 2 || !dims || dims[0] == 0 || dims[0] != dims[1] || dims[0] > (1u << 16))
      return fail(CAFXG_E_INTERFACE_MISMATCH,
                  "spawn: matrix_multiply takes dims {size, size}");
  } else {
    return fail(CAFXG_E_UNKNOWN_TYPE, "spawn: no kernel named '%s'", kernel_name);
  }
  auto* a = new cafxg_actor;
  a->ctx = ctx;
  a->kernel = k;
  a->ndims = std::min<size_t>(ndims, 3);
  for (size_t i = 0; i < a->ndims; ++i)
    a->dims[i] = dims[i];
  *out = a;
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_spawn: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_spawn: unknown exception");
}

static int actor_check(cafxg_actor* a, const void* const* in, const size_t* in_bytes,
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

int cafxg_fnv1a_u32_device(cafxg_ctx* ctx, int device, const uint32_t* cells, uint64_t n,
                           uint64_t seed, uint64_t* hash, void* stream) try {
  if (!ctx || !hash || device < 0 || device >= (int)ctx->devs.size() || (n && !cells))
    return fail(CAFXG_E_CONFIG, "fnv1a_u32_device: bad argument");
  Device* d = ctx->devs[device].get();
  cudaSetDevice(d->ordinal);
  cudaStream_t s = stream ? (cudaStream_t)stream : d->compute;
  void* scratch = nullptr;
  uint64_t* dhash = nullptr;
  CAFXG_CUDA_TRY(cudaMallocAsync(&scratch, fnv_scratch_bytes(n, d->sms), s));
  CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dhash, sizeof(uint64_t), s));
  int launches = 0;
  int e = fnv_launch(cells, n, seed, dhash, scratch, d->sms, s, &launches);
  if (e != 0)
    return cuda_status((cudaError_t)e, "fnv launch");
  ctx->st_launches += launches;
  CAFXG_CUDA_TRY(cudaMemcpyAsync(hash, dhash, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  CAFXG_CUDA_TRY(cudaFreeAsync(scratch, s));
  CAFXG_CUDA_TRY(cudaFreeAsync(dhash, s));
  CAFXG_CUDA_TRY(cudaStreamSynchronize(s));
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_fnv1a_u32_device: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_fnv1a_u32_device: unknown exception");
}

// run_mandelbrot(size, max_iter) (bench.cpp:481-505) on the context's devices:
// the reference-mode image (fp64, corner sampling, [-1.5,0.5]x[-1,1]) is
// computed in HBM in contiguous row blocks per device, each device hashes its
// block with the segment-table FNV (fnv.cu), and the per-device hashes are
// chained on the host in row order: the checksum is the reference's
// collector hash (bench.cpp:329-331) without moving the image off the GPUs.
int cafxg_run_mandelbrot(cafxg_ctx* ctx, uint32_t size, uint32_t max_iter, uint64_t* checksum,
                         double* wall_ms) try {
  if (!ctx || !checksum || size == 0)
    return fail(CAFXG_E_CONFIG, "run_mandelbrot: bad argument");
  auto t0 = std::chrono::steady_clock::now();
  const size_t G = std::min<size_t>(ctx->devs.size(), size);
  std::vector<uint32_t*> img(G, nullptr);
  std::vector<uint64_t*> dh(G, nullptr);
  std::vector<uint64_t> hh(G, 0);
  std::vector<uint32_t> r0(G + 1);
  for (size_t g = 0; g <= G; ++g)
    r0[g] = (uint32_t)((uint64_t)size * g / G);
  // Per device: its block of rows in one escape launch, then the seed-
  // independent FNV pass 1 (per-segment low-byte tables, the bulk of the
  // hash) -- in parallel on every device. Then the cheap seeded passes run
  // device after device, each block seeded with the previous block's hash
  // (FNV is sequential). Overlapping pass 1 with the image on one device
  // was tried and is slower.
  std::vector<void*> scratch(G, nullptr);
  for (size_t g = 0; g < G; ++g) {
    Device* d = ctx->devs[g].get();
    cudaSetDevice(d->ordinal);
    uint64_t rows = r0[g + 1] - r0[g];
    uint64_t n = rows * size;
    CAFXG_CUDA_TRY(cudaMallocAsync((void**)&img[g], n * 4 + 16, d->compute));
    CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dh[g], 8, d->compute));
    CAFXG_CUDA_TRY(cudaMallocAsync(&scratch[g], fnv_scratch_bytes(n, d->sms), d->compute));
    cafxg_mandel_desc t{};
    t.x0 = -1.5; t.x1 = 0.5; t.y0 = -1.0; t.y1 = 1.0;
    t.width = t.height = size;
    t.row0 = r0[g];
    t.nrows = (uint32_t)rows;
    t.ncols = size;
    t.max_iter = max_iter;
    t.precision = CAFXG_FP64;
    t.sampling = CAFXG_CORNER;
    CAFXG_TRY(validate_mandel(t));
    MTile m;
    fill_mtile(m, t, 0, 0);
    CAFXG_TRY(launch_mandel(ctx, d, img[g], {m}, tile_chunks(t.nrows, t.ncols, CAFXG_FP64), CAFXG_FP64,
                            max_iter, use_exact(ctx, t), n, d->compute));
    uint64_t seg_cells = 0;
    uint32_t nseg = 0;
    fnv_segments(n, d->sms, &seg_cells, &nseg);
    int e = fnv_lowbyte_launch(img[g], n, 0, nseg, scratch[g], d->sms, d->compute);
    if (e != 0)
      return cuda_status((cudaError_t)e, "fnv pass-1 launch");
    ctx->st_launches++;
  }
  // the seeded passes, block after block
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t g = 0; g < G; ++g) {
    Device* d = ctx->devs[g].get();
    cudaSetDevice(d->ordinal);
    uint64_t n = (uint64_t)(r0[g + 1] - r0[g]) * size;
    int launches = 0;
    int e = fnv_finish_launch(img[g], n, h, dh[g], scratch[g], d->sms, d->compute, &launches);
    if (e != 0)
      return cuda_status((cudaError_t)e, "fnv launch");
    ctx->st_launches += launches;
    CAFXG_CUDA_TRY(cudaMemcpyAsync(&hh[g], dh[g], 8, cudaMemcpyDeviceToHost, d->compute));
    CAFXG_CUDA_TRY(cudaStreamSynchronize(d->compute));
    h = hh[g];
  }
  for (size_t g = 0; g < G; ++g) {
    Device* d = ctx->devs[g].get();
    cudaSetDevice(d->ordinal);
    cudaFreeAsync(img[g], d->compute);
    cudaFreeAsync(dh[g], d->compute);
    cudaFreeAsync(scratch[g], d->compute);
  }
  *checksum = h;
  if (wall_ms)
    *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                   .count();
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_run_mandelbrot: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_run_mandelbrot: unknown exception");
}

int cafxg_get_stats(cafxg_ctx* ctx, cafxg_stats* out) {
  if (!ctx || !out)
    return fail(CAFXG_E_CONFIG, "get_stats: null argument");
  out->requests = ctx->st_requests.load();
  out->batches = ctx->st_batches.load();
  out->kernel_launches = ctx->st_launches.load();
  out->h2d_bytes = ctx->st_h2d.load();
  out->d2h_bytes = ctx->st_d2h.load();
  out->max_batch = ctx->st_max_batch.load();
  out->direct_batches = ctx->st_direct.load();
  return CAFXG_OK;
}

}  // extern "C"
