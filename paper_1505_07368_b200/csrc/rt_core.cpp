// libcafxg.so host runtime, core: error context, pinned pool, device
// completion threads, stream ordering helpers and the context lifecycle
// (cafxg_open / cafxg_close) of the C ABI in include/cafxg.h.
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
#include "runtime_internal.hpp"

namespace cafxg {

// ---- error context -----------------------------------------------------------

thread_local std::string t_last_error;

void set_last_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_last_error = buf;
}

void clear_last_error() { t_last_error.clear(); }

// True when [p, p+bytes) is page-locked host memory the device can address
// (our pool, cudaHostRegister'ed or torch pin_memory buffers).
bool host_is_pinned(const void* p, size_t bytes) {
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

// Host clock for CAFXG_TRACE timelines (ms since first use).
double trace_now_ms() {
  static const auto t0 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

void note_max_batch(cafxg_ctx* ctx, uint64_t n) {
  uint64_t cur = ctx->st_max_batch.load();
  while (n > cur && !ctx->st_max_batch.compare_exchange_weak(cur, n)) {
  }
}

// Backend threads (dispatcher, completion) get a higher scheduling weight
// than client threads when the process may raise it (best effort): under a
// request storm, clients outnumber cores, and a starved completion thread
// leaves the device idle with finished batches counted as in flight.
void raise_priority() {
  setpriority(PRIO_PROCESS, (id_t)syscall(SYS_gettid), -10);
}

void completion_loop(cafxg_ctx* ctx, Device* d) {
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
    int status = c.status;
    if (c.ev) {
      cudaError_t e = cudaEventSynchronize(c.ev);
      const uint64_t nth = ctx->completions.fetch_add(1) + 1;
      if (e == cudaSuccess && ctx->simulate_loss_at && nth >= ctx->simulate_loss_at)
        e = cudaErrorLaunchFailure;  // CAFXG_SIMULATE_DEVICE_LOSS (tests)
      if (e != cudaSuccess) {
        status = cuda_status(e, "device work failed");
        mark_lost(ctx, e, "device work failed");
      }
    }
    {
      NvtxRange nvtx_range("cafxg.complete");
      run_guarded("completion callback", [&] { c.fn(status); });
    }
    if (c.ev) {
      std::lock_guard<std::mutex> lk(d->cq_mu);
      d->ev_free.push_back(c.ev);
    }
    d->inflight.fetch_sub(1);
    {
      std::lock_guard<std::mutex> lk(ctx->sync_mu);
      ++ctx->completed;
    }
    ctx->sync_cv.notify_all();
    // The dispatcher's wait predicate reads `inflight`: taking its mutex
    // between the decrement and the notify keeps the notify from falling
    // between its predicate check and its sleep (a lost wakeup stalled a
    // closed-loop storm with every device at its in-flight cap).
    { std::lock_guard<std::mutex> lk(ctx->disp_mu); }
    ctx->disp_cv.notify_all();
  }
}

// Errors after which the CUDA context of the device is unusable: every later
// call fails with the same error until the process exits.
static bool sticky(cudaError_t e) {
  switch (e) {
    case cudaErrorIllegalAddress:
    case cudaErrorLaunchFailure:
    case cudaErrorHardwareStackError:
    case cudaErrorIllegalInstruction:
    case cudaErrorMisalignedAddress:
    case cudaErrorInvalidAddressSpace:
    case cudaErrorInvalidPc:
    case cudaErrorECCUncorrectable:
    case cudaErrorAssert:
    case cudaErrorLaunchTimeout:
    case cudaErrorContextIsDestroyed:
    case cudaErrorDevicesUnavailable:
      return true;
    default:
      return false;
  }
}

void mark_lost(cafxg_ctx* ctx, cudaError_t e, const char* where) {
  if (!sticky(e) || ctx->lost.load())
    return;
  {
    std::lock_guard<std::mutex> g(ctx->lost_mu);
    ctx->lost_why = std::string(where) + ": " + cudaGetErrorName(e);
  }
  ctx->lost.store(true);
  { std::lock_guard<std::mutex> lk(ctx->disp_mu); }  // see completion_loop
  ctx->disp_cv.notify_all();
}

int check_alive(cafxg_ctx* ctx) {
  if (!ctx->lost.load(std::memory_order_relaxed))
    return CAFXG_OK;
  std::lock_guard<std::mutex> g(ctx->lost_mu);
  return fail(CAFXG_E_DOWN, "context lost after a sticky device error (%s)",
              ctx->lost_why.c_str());
}

// Backend threads never let an exception escape (it would terminate the
// process): a throwing callback or task is reported on stderr and skipped.
void run_guarded(const char* what, const std::function<void()>& fn) {
  try {
    fn();
  } catch (const std::exception& ex) {
    fprintf(stderr, "cafxg: %s threw: %s\n", what, ex.what());
  } catch (...) {
    fprintf(stderr, "cafxg: %s threw a non-standard exception\n", what);
  }
}

void issuer_loop(Device* d) {
  cudaSetDevice(d->ordinal);
  while (true) {
    std::function<void()> fn;
    {
      std::unique_lock<std::mutex> lk(d->iq_mu);
      d->iq_cv.wait(lk, [&] { return d->iq_stop || !d->iq.empty(); });
      if (d->iq.empty())
        return;
      fn = std::move(d->iq.front());
      d->iq.pop_front();
    }
    run_guarded("issue task", fn);
  }
}

void issue_async(cafxg_ctx* ctx, Device* d, std::function<void()> fn) {
  ctx->issuing.fetch_add(1);
  {
    std::lock_guard<std::mutex> lk(d->iq_mu);
    d->iq.push_back([ctx, fn = std::move(fn)] {
      fn();
      ctx->issuing.fetch_sub(1);
      ctx->sync_cv.notify_all();
    });
  }
  d->iq_cv.notify_one();
}

// Records an event on `stream` and hands `fn` to the device's completion
// thread. Caller holds d->submit_mu (so records stay in stream order).
__global__ void trap_kernel() { asm volatile("trap;"); }

void push_completion(cafxg_ctx* ctx, Device* d, cudaStream_t stream,
                     std::function<void(int)> fn) {
  if (ctx->inject_trap_at && ctx->pushes.fetch_add(1) + 1 == ctx->inject_trap_at) {
    trap_kernel<<<1, 32, 0, stream>>>();
    if (ctx->inject_trap_sync)
      cudaStreamSynchronize(stream);
  }
  cudaEvent_t ev = nullptr;
  {
    std::lock_guard<std::mutex> lk(d->cq_mu);
    if (!d->ev_free.empty()) {
      ev = d->ev_free.back();
      d->ev_free.pop_back();
    }
  }
  cudaError_t e = cudaSuccess;
  if (!ev)
    e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess)
    e = cudaEventRecord(ev, stream);
  int status = CAFXG_OK;
  if (e != cudaSuccess) {
    // No event: the callback still runs, on the completion thread, after
    // whatever is queued on the stream (best effort on a broken context) and
    // with the error. Dropping it would leave the request's waiter asleep.
    status = cuda_status(e, "completion event");
    mark_lost(ctx, e, "completion event");
    cudaStreamSynchronize(stream);
    cudaGetLastError();
    if (ev) {
      std::lock_guard<std::mutex> lk(d->cq_mu);
      d->ev_free.push_back(ev);
    }
    ev = nullptr;
  }
  {
    std::lock_guard<std::mutex> lk(ctx->sync_mu);
    ++ctx->submitted;
  }
  d->inflight.fetch_add(1);
  {
    std::lock_guard<std::mutex> lk(d->cq_mu);
    d->cq.push_back(Completion{ev, std::move(fn), status});
  }
  d->cq_cv.notify_one();
}

// Host -> device copy of small descriptor arrays through the device's pinned
// staging ring, so the call never waits for earlier work on `stream`.
int upload(Device* d, void* dst, const void* src, size_t bytes, cudaStream_t stream) {
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

bool trace_on() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}

int stream_after(cudaStream_t b, cudaStream_t a) {
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
int stream_after_pooled(Device* d, cudaStream_t b, cudaStream_t a) {
  if (!d->order_ev)
    CAFXG_CUDA_TRY(cudaEventCreateWithFlags(&d->order_ev, cudaEventDisableTiming));
  CAFXG_CUDA_TRY(cudaEventRecord(d->order_ev, a));
  CAFXG_CUDA_TRY(cudaStreamWaitEvent(b, d->order_ev, 0));
  return CAFXG_OK;
}

cudaEvent_t pooled_event(Device* d) {
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

void Waiter::cb(void* u, int s) {
  auto* w = static_cast<Waiter*>(u);
  std::lock_guard<std::mutex> g(w->mu);
  w->fired = true;
  w->status = s;
  if (s != CAFXG_OK)
    w->err = t_last_error;
  w->cv.notify_all();
}

int Waiter::wait() {
  std::unique_lock<std::mutex> lk(mu);
  cv.wait(lk, [&] { return fired; });
  if (status != CAFXG_OK)
    set_last_error("%s", err.c_str());
  return status;
}

}  // namespace cafxg

using namespace cafxg;

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
    const char* p2p = getenv("CAFXG_SGEMM_P2P");
    ctx->p2p_off = p2p && p2p[0] == '0';
    const char* vd = getenv("CAFXG_VIRTUAL_DEVICES");
    int vcount = vd ? atoi(vd) : 0;
    if (vcount > 1 && ords.size() == 1) {
      ords.assign(std::min(vcount, 64), ords[0]);
      ctx->virtual_devs = true;
    }
    for (int i : ords) {
      auto d = std::make_unique<Device>();
      d->ordinal = i;
      d->index = (int)ctx->devs.size();
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
      // complete before any launch on the non-blocking streams reads a cursor
      CAFXG_CUDA_TRY(cudaStreamSynchronize(0));
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
    if (const char* sl = getenv("CAFXG_SIMULATE_DEVICE_LOSS"))
      ctx->simulate_loss_at = (uint64_t)std::max(0, atoi(sl));
    if (const char* t = getenv("CAFXG_INJECT_TRAP"))
      ctx->inject_trap_at = (uint64_t)std::max(0, atoi(t));
    if (const char* t = getenv("CAFXG_INJECT_TRAP_SYNC"))
      ctx->inject_trap_sync = t[0] == '1';
    cafxg_ctx* c = ctx.release();
    for (auto& d : c->devs) {
      d->completer = std::thread(completion_loop, c, d.get());
      if (c->devs.size() > 1)
        d->issuer = std::thread(issuer_loop, d.get());
    }
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
  while (!(ctx->completed == ctx->submitted && ctx->actor_open.load() == 0 &&
           ctx->issuing.load() == 0))
    ctx->sync_cv.wait_for(lk, std::chrono::milliseconds(1));
  return CAFXG_OK;
}

int cafxg_close(cafxg_ctx* ctx) try {
  if (!ctx)
    return CAFXG_OK;
  if (trace_on() || getenv("CAFXG_STATS"))
    fprintf(stderr, "cafxg: pinned pool: %llu driver allocations\n",
            (unsigned long long)ctx->pinned.new_allocs());
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
  // issuers drain their queues first: what they issue reports through the
  // completion threads below
  for (auto& d : ctx->devs) {
    {
      std::lock_guard<std::mutex> lk(d->iq_mu);
      d->iq_stop = true;
    }
    d->iq_cv.notify_all();
    if (d->issuer.joinable())
      d->issuer.join();
  }
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
    for (auto ev : d->sched_ev)
      if (ev)
        cudaEventDestroy(ev);
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

int cafxg_ctx_status(cafxg_ctx* ctx) {
  if (!ctx)
    return fail(CAFXG_E_CONFIG, "ctx_status: null ctx");
  return check_alive(ctx);
}

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
  out->nccl_collectives = ctx->st_nccl.load();
  out->peer_gemms = ctx->st_p2p.load();
  out->devices_used = ctx->st_dev_used.load();
  return CAFXG_OK;
}

}  // extern "C"
