// Internal declarations shared by the host runtime units of libcafxg.so
// (rt_core.cpp, rt_mandel.cpp, rt_sgemm.cpp, rt_actor.cpp): the pinned pool,
// devices, the context, request joins and the cross-unit helpers.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

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

// context string of the last failure on this thread (cafxg_last_error)
extern thread_local std::string t_last_error;

// ---- pinned host pool -----------------------------------------------------------
// Page-locked, portable, device-mapped buffers cached by power-of-two size
// class. Reply buffers that live here are written by DMA or by the reply
// scatter kernel directly. Classes up to kSlabClassMax are carved out of
// 64 MB slabs: one driver call per slab instead of one per buffer (a storm
// of 102,400 outstanding 16 KB replies made ~100K cudaHostAlloc calls, which
// serialise on the driver lock against the dispatcher's launches and copies).
class PinnedPool {
 public:
  static constexpr size_t kSlabBytes = 64ull << 20;
  static constexpr size_t kSlabClassMax = 1ull << 20;

  ~PinnedPool() {
    std::lock_guard<std::mutex> g(mu_);
    for (void* p : slabs_)
      cudaFreeHost(p);
    for (void* p : large_)
      cudaFreeHost(p);
  }

  void* alloc(size_t bytes) {
    const size_t cls = size_class(bytes);
    {
      std::lock_guard<std::mutex> g(mu_);
      if (void* p = take_locked(cls))
        return p;
    }
    // driver calls outside the lock: a pinned allocation takes milliseconds
    // (a 1 GiB image ~0.1 s) and completion threads free buffers meanwhile
    if (cls > kSlabClassMax) {
      void* p = nullptr;
      new_allocs_.fetch_add(1, std::memory_order_relaxed);
      if (cudaHostAlloc(&p, cls, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      std::lock_guard<std::mutex> g(mu_);
      large_.push_back(p);
      add_range(p, cls);
      live_[p] = cls;
      return p;
    }
    void* s = nullptr;
    new_allocs_.fetch_add(1, std::memory_order_relaxed);
    if (cudaHostAlloc(&s, kSlabBytes, cudaHostAllocPortable | cudaHostAllocMapped) !=
        cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    std::lock_guard<std::mutex> g(mu_);
    slabs_.push_back(s);
    add_range(s, kSlabBytes);
    // (a slab another thread installed meanwhile keeps its tail unused)
    slab_ = (uint8_t*)s;
    slab_used_ = 0;
    return take_locked(cls);
  }

  // driver allocations so far (CAFXG_STATS=1 prints them at close)
  uint64_t new_allocs() const { return new_allocs_.load(std::memory_order_relaxed); }

  bool free(void* p) {
    std::lock_guard<std::mutex> g(mu_);
    auto it = live_.find(p);
    if (it == live_.end())
      return false;
    free_[it->second].push_back(p);
    live_.erase(it);
    return true;
  }

  // [p, p+bytes) inside one pool slab or buffer (no driver call). Every client
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
  // a cached buffer of class cls, or one carved from the current slab
  void* take_locked(size_t cls) {
    auto it = free_.find(cls);
    if (it != free_.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      live_[p] = cls;
      return p;
    }
    if (cls <= kSlabClassMax && slab_ && slab_used_ + cls <= kSlabBytes) {
      void* p = slab_ + slab_used_;  // classes are multiples of 4 KB: page-aligned
      slab_used_ += cls;
      live_[p] = cls;
      return p;
    }
    return nullptr;
  }
  void add_range(void* p, size_t bytes) {
    std::unique_lock<std::shared_mutex> w(ranges_mu_);
    ranges_[(uintptr_t)p] = bytes;
  }
  std::mutex mu_;
  std::atomic<uint64_t> new_allocs_{0};
  std::unordered_map<void*, size_t> live_;
  std::map<size_t, std::vector<void*>> free_;
  std::vector<void*> slabs_, large_;  // what the driver allocated
  uint8_t* slab_ = nullptr;           // the slab small classes are carved from
  size_t slab_used_ = 0;
  mutable std::shared_mutex ranges_mu_;
  std::map<uintptr_t, size_t> ranges_;  // every slab and large buffer
  // unique per pool instance (never reused), so a thread-local cache entry of
  // a closed context can never match a later one
  static inline std::atomic<uint64_t> next_id_{1};
  const uint64_t id_ = next_id_.fetch_add(1);
};

// True when [p, p+bytes) is page-locked host memory the device can address
// (our pool, cudaHostRegister'ed or torch pin_memory buffers).
bool host_is_pinned(const void* p, size_t bytes);

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
  cudaEvent_t ev;  // null: no event could be recorded, `status` is the outcome
  std::function<void(int)> fn;
  int status = 0;
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
// Actor requests of at least this many pixels are not batched: they go the
// host-request way (row bands over every device, overlapped waves).
constexpr uint64_t kLargeActorPx = 1ull << 20;
constexpr int kUpSlots = 16;
constexpr size_t kUpSlotBytes = 2u << 20;

struct Device {
  int ordinal = 0;
  int index = 0;  // position in the context's device list
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
  // issuer thread (multi-device contexts): the per-device share of a request
  // is issued here, so every device's first wave starts at once instead of
  // after the previous devices' host-side issue (~20 us per wave)
  std::mutex iq_mu;
  std::condition_variable iq_cv;
  std::deque<std::function<void()>> iq;
  bool iq_stop = false;
  std::thread issuer;

  // Self-resetting scheduler slots: slot i is free again once the launch that
  // last used it has finished; sched_acquire orders `stream` after that launch
  // (two launches 1024 slots apart on different streams would
  // otherwise share one cursor).
  std::mutex sched_mu;
  cudaEvent_t sched_ev[kSchedSlots] = {};
  uint32_t sched_acquire(cudaStream_t stream) {
    const uint32_t i = sched_next.fetch_add(1, std::memory_order_relaxed) % kSchedSlots;
    std::lock_guard<std::mutex> g(sched_mu);
    if (sched_ev[i])
      cudaStreamWaitEvent(stream, sched_ev[i], 0);
    return i;
  }
  void sched_release(uint32_t i, cudaStream_t stream) {
    std::lock_guard<std::mutex> g(sched_mu);
    if (!sched_ev[i] && cudaEventCreateWithFlags(&sched_ev[i], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      sched_ev[i] = nullptr;
      return;
    }
    cudaEventRecord(sched_ev[i], stream);
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
  std::atomic<uint64_t> st_nccl{0};      // NCCL collectives issued (B all-gathers)
  std::atomic<uint64_t> st_p2p{0};       // multi-device GEMMs reading B's slices in place
  std::atomic<uint64_t> st_dev_used{0};  // bit i: context device i ran a kernel
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
  std::atomic<uint64_t> issuing{0};     // issuer tasks queued or running (cafxg_sync)
  // reply-callback threads (finish_batch)
  std::mutex cb_mu;
  std::condition_variable cb_cv;
  std::deque<std::function<void()>> cb_q;
  bool cb_stop = false;
  std::vector<std::thread> cb_threads;
  bool force_exact = false;  // CAFXG_EXACT_STEP=1: always the 8-op step
  // A sticky CUDA error (the CUDA context of a device is unusable) makes the
  // whole context lost: later submissions fail at once with CAFXG_E_DOWN and
  // cafxg_ctx_status reports it, so adapters can terminate their actors
  // (abstract_actor.cpp:108-134) instead of failing every request one by one.
  std::atomic<bool> lost{false};
  std::mutex lost_mu;
  std::string lost_why;
  // CAFXG_SIMULATE_DEVICE_LOSS=<n> (read at cafxg_open; tests only): the n-th
  // completion of the context reports cudaErrorLaunchFailure, as a real
  // sticky fault would, without faulting the GPU
  uint64_t simulate_loss_at = 0;
  // CAFXG_INJECT_TRAP=n (tests): a trapping kernel is queued ahead of the
  // n-th completion event, a real sticky device fault; with
  // CAFXG_INJECT_TRAP_SYNC=1 the fault is waited for first, so recording the
  // completion event itself fails
  uint64_t inject_trap_at = 0;
  bool inject_trap_sync = false;
  std::atomic<uint64_t> pushes{0};
  std::atomic<uint64_t> completions{0};
  // CAFXG_VIRTUAL_DEVICES=V: V context devices on one physical GPU (own
  // streams, scheduler ring and completion thread each) so the multi-device
  // split/join logic runs on a single-GPU box; B is then replicated by
  // device-to-device copies instead of NCCL (which rejects duplicate GPUs)
  bool virtual_devs = false;
  // NCCL communicators for multi-device sgemm (one per device)
  std::mutex nccl_mu;
  bool nccl_failed = false;
  bool p2p_off = false;  // CAFXG_SGEMM_P2P=0 at open: B exchanged by NCCL, not read in place
  int p2p_state = 0;  // peer access between every pair of GPUs: 0 unknown, 1 yes, -1 no
  NcclApi nccl;
  std::vector<ncclComm_t> comms;
};

namespace cafxg {

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

struct SubTile {
  cafxg_mandel_desc d;  // row0/nrows narrowed; out_offset = host offset
  uint64_t pixels;
};

// records that context device `d` has run a kernel (cafxg_stats::devices_used)
inline void mark_used(cafxg_ctx* ctx, const Device* d) {
  ctx->st_dev_used.fetch_or(1ull << (d->index & 63), std::memory_order_relaxed);
}

// NVTX range over a host-side scope (request submission, batches, reply
// callbacks): visible in Nsight Systems / ncu timelines, a no-op without a tool
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---- rt_core.cpp ----
// runs fn, reporting (not propagating) an exception: backend threads
void run_guarded(const char* what, const std::function<void()>& fn);
// runs `fn` on device d's issuer thread (multi-device contexts)
void issue_async(cafxg_ctx* ctx, Device* d, std::function<void()> fn);
void issuer_loop(Device* d);
// marks the context lost after a sticky CUDA error (see cafxg_ctx::lost)
void mark_lost(cafxg_ctx* ctx, cudaError_t e, const char* where);
// CAFXG_E_DOWN (with the loss recorded as the error context) once lost
int check_alive(cafxg_ctx* ctx);
double trace_now_ms();
bool trace_on();
void note_max_batch(cafxg_ctx* ctx, uint64_t n);
void raise_priority();
void completion_loop(cafxg_ctx* ctx, Device* d);
// Records an event on `stream` and hands `fn` to the device's completion
// thread. Caller holds d->submit_mu (so records stay in stream order).
// Runs fn(status) on the device's completion thread once the work queued on
// `stream` so far has finished. fn is called exactly once on every path: when
// not even an event can be recorded (a dead context), the stream is drained
// here and fn receives the error.
void push_completion(cafxg_ctx* ctx, Device* d, cudaStream_t stream, std::function<void(int)> fn);
// Host -> device copy of small descriptor arrays through the device's pinned
// staging ring, so the call never waits for earlier work on `stream`.
int upload(Device* d, void* dst, const void* src, size_t bytes, cudaStream_t stream);
int stream_after(cudaStream_t b, cudaStream_t a);  // b waits for a's work so far
int stream_after_pooled(Device* d, cudaStream_t b, cudaStream_t a);
cudaEvent_t pooled_event(Device* d);

// Blocking wait on a completion callback (the blocking C-ABI wrappers).
struct Waiter {
  std::mutex mu;
  std::condition_variable cv;
  bool fired = false;
  int status = CAFXG_OK;
  std::string err;
  static void cb(void* u, int s);
  int wait();
};

// ---- rt_mandel.cpp ----
int validate_mandel(const cafxg_mandel_desc& t);
bool use_exact(cafxg_ctx* ctx, const cafxg_mandel_desc& t);
uint32_t tile_chunks(uint32_t nrows, uint32_t ncols, uint32_t precision);
void fill_mtile(MTile& m, const cafxg_mandel_desc& d, uint64_t out_off, uint32_t chunk_begin);
bool direct_reply_enabled();
int launch_mandel(cafxg_ctx* ctx, Device* d, uint32_t* out_base,
                  const std::vector<MTile>& tiles_in, uint32_t total_chunks,
                  int precision, uint32_t max_iter, bool exact,
                  uint64_t pixels, cudaStream_t stream,
                  uint32_t* direct_counters = nullptr,
                  const cafxg_tuning* tune = nullptr);
std::vector<std::vector<SubTile>> plan_mandel(const cafxg_mandel_desc* tiles, size_t n, size_t ndev);
int mandel_submit_impl(cafxg_ctx* ctx, const cafxg_mandel_desc* tiles, size_t n,
                       uint32_t* host_out, cafxg_done_fn done, void* user,
                       const cafxg_tuning* tune = nullptr);

// ---- rt_sgemm.cpp ----
int sgemm_submit_impl(cafxg_ctx* ctx, const cafxg_sgemm_desc* desc, const float* A,
                      const float* B, float* C, cafxg_done_fn done, void* user);

// ---- rt_actor.cpp ----
void dispatcher_loop(cafxg_ctx* ctx);
void callback_loop(cafxg_ctx* ctx);

}  // namespace cafxg
