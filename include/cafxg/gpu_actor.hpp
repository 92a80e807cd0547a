// gpu_actor.hpp -- the CAF side of the drop-in: a compute actor on the cafx
// runtime's own seam, backed by libcafxg.so (include/cafxg.h).
//
// Header-only. Compile inside a cafx program with the reference's include/
// and this repo's include/ on the include path, link libcafxg.so.
//
//   cafx::actor_system sys;
//   cafxg_ctx* ctx; cafxg_open(0, &ctx);
//   auto mm = cafxg::spawn_gpu(sys, ctx, "matrix_multiply", {size, size});
//   // == spawn_cl<float*(float*,float*)>(src, "matrix_multiply", {size, size})
//   //    (PAPER.md:357-361): request (f32vec, f32vec) -> reply f32vec
//   auto mb = cafxg::spawn_gpu(sys, ctx, "mandelbrot", {});
//   //    request (cafxg::mandel_tiles) -> reply u32vec
//
// What it implements, against the reference runtime:
//  * `enqueue` (abstract_actor.hpp:36) may be called from any thread; it
//    decodes the request and hands it to cafxg_actor_enqueue (never blocks on
//    the device) -- the remote_proxy precedent (middleman.cpp:115-146);
//  * replies follow local_actor::respond (local_actor.cpp:319-329): requests
//    get `mid | 1<<63` after drop_pending_request, async sends with a sender
//    get a plain reply; failures are a 1-element `error{errc, context}`
//    message (scoped_actor.cpp:209-211). Replies are posted from libcafxg's
//    completion thread, never from a scheduler worker;
//  * exit signals: a hard kill (actor_system.cpp:243-258) or a non-normal exit
//    quits the backend actor, `finalize`s (monitors, links, request_down for
//    pending requesters, abstract_actor.cpp:108-134) and unregisters, so
//    ~actor_system does not wait forever (actor_system.cpp:21-30);
//  * buffer types are registered with wire codecs (type_registry.hpp:74-80),
//    so middleman::publish can serve a GPU actor to remote nodes;
//  * reply relay: a reply leaves libcafxg's completion thread through a
//    lock-free per-actor queue drained by a job on the cafx scheduler
//    (actor_system::schedule_job, scheduler.hpp:266-274), so the requesters
//    are made runnable from a worker thread (its own deque) and a whole batch
//    of replies costs one external enqueue instead of one each. External
//    enqueues contend with the idle workers' steal sweeps over the deque
//    mutexes (scheduler.hpp:374-402): delivering from a foreign thread cost
//    ~15 us per reply against ~2.5-8 us relayed (a CPU probe of the pattern,
//    DESIGN.md §5).
#pragma once

#include <atomic>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <memory>
#include <new>
#include <type_traits>
#include <string>
#include <utility>
#include <vector>

#include "cafx/abstract_actor.hpp"
#include "cafx/actor_system.hpp"
#include "cafx/detail/wire.hpp"
#include "cafx/envelope.hpp"
#include "cafx/error.hpp"
#include "cafx/handle.hpp"
#include "cafx/interface.hpp"
#include "cafx/message.hpp"
#include "cafx/resumable.hpp"
#include "cafx/type_registry.hpp"
#include "cafxg.h"

namespace cafxg {

/// Allocator of the buffer types. Default-constructed it is the plain heap
/// (wire decoding, user-built requests). Bound to a context it takes memory
/// from the context's pinned, device-mapped pool (cafxg_host_alloc) and
/// leaves elements uninitialised: the adapter sizes reply vectors with it, so
/// the kernel writes counts straight into the vector the reply message owns
/// (no zero-fill, no staging copy). Such a vector must not outlive its
/// context. Users may bind it too, to make request payloads DMA-able.
template <class T>
struct host_allocator {
  using value_type = T;
  using propagate_on_container_copy_assignment = std::true_type;
  using propagate_on_container_move_assignment = std::true_type;
  using propagate_on_container_swap = std::true_type;
  cafxg_ctx* ctx = nullptr;

  host_allocator() noexcept = default;
  explicit host_allocator(cafxg_ctx* c) noexcept : ctx(c) {}
  template <class U>
  host_allocator(const host_allocator<U>& o) noexcept : ctx(o.ctx) {}

  T* allocate(size_t n) {
    if (!ctx)
      return std::allocator<T>{}.allocate(n);
    void* p = nullptr;
    if (cafxg_host_alloc(ctx, n * sizeof(T), &p) != CAFXG_OK)
      throw std::bad_alloc{};
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t n) noexcept {
    if (!ctx)
      std::allocator<T>{}.deallocate(p, n);
    else
      cafxg_host_free(ctx, p);
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    if constexpr (sizeof...(Args) == 0) {
      if (ctx) {
        ::new (static_cast<void*>(p)) U;  // default-init: the device fills it
        return;
      }
    }
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
  template <class U>
  bool operator==(const host_allocator<U>& o) const noexcept { return ctx == o.ctx; }
};

using f32vec = std::vector<float, host_allocator<float>>;
using u32vec = std::vector<uint32_t, host_allocator<uint32_t>>;

/// Request payload of the "mandelbrot" kernel: one or more tiles; the reply
/// is their counts packed in order.
struct mandel_tiles {
  std::vector<cafxg_mandel_desc> tiles;
  bool operator==(const mandel_tiles& o) const {
    return tiles.size() == o.tiles.size() &&
           std::memcmp(tiles.data(), o.tiles.data(),
                       tiles.size() * sizeof(cafxg_mandel_desc)) == 0;
  }
};

namespace codec {

inline void put_f64(cafx::byte_buffer& b, double x) {
  cafx::detail::put_u64(b, cafx::detail::double_bits(x));
}
inline double get_f64(cafx::detail::reader& r) {
  uint64_t bits = r.u64();
  double x;
  std::memcpy(&x, &bits, 8);
  return x;
}

inline void enc_f32vec(const std::any& v, cafx::byte_buffer& out) {
  const auto& x = *std::any_cast<f32vec>(&v);
  cafx::detail::put_u32(out, static_cast<uint32_t>(x.size()));
  for (float f : x)
    cafx::detail::put_u32(out, cafx::detail::float_bits(f));
}
inline std::any dec_f32vec(cafx::detail::reader& in) {
  f32vec x(in.u32());
  for (auto& f : x) {
    uint32_t bits = in.u32();
    std::memcpy(&f, &bits, 4);
  }
  in.expect_done();
  return std::any{std::move(x)};
}
inline void enc_u32vec(const std::any& v, cafx::byte_buffer& out) {
  const auto& x = *std::any_cast<u32vec>(&v);
  cafx::detail::put_u32(out, static_cast<uint32_t>(x.size()));
  for (uint32_t c : x)
    cafx::detail::put_u32(out, c);  // big-endian cells, like pack_row
}
inline std::any dec_u32vec(cafx::detail::reader& in) {
  u32vec x(in.u32());
  for (auto& c : x)
    c = in.u32();
  in.expect_done();
  return std::any{std::move(x)};
}
inline void enc_tiles(const std::any& v, cafx::byte_buffer& out) {
  const auto& x = *std::any_cast<mandel_tiles>(&v);
  cafx::detail::put_u32(out, static_cast<uint32_t>(x.tiles.size()));
  for (const auto& t : x.tiles) {
    put_f64(out, t.x0);
    put_f64(out, t.x1);
    put_f64(out, t.y0);
    put_f64(out, t.y1);
    for (uint32_t u : {t.width, t.height, t.row0, t.nrows, t.col0, t.ncols,
                       t.max_iter, t.precision, t.sampling})
      cafx::detail::put_u32(out, u);
    cafx::detail::put_u64(out, t.out_offset);
  }
}
inline std::any dec_tiles(cafx::detail::reader& in) {
  mandel_tiles x;
  x.tiles.resize(in.u32());
  for (auto& t : x.tiles) {
    t = cafxg_mandel_desc{};
    t.x0 = get_f64(in);
    t.x1 = get_f64(in);
    t.y0 = get_f64(in);
    t.y1 = get_f64(in);
    uint32_t* f[] = {&t.width, &t.height, &t.row0, &t.nrows, &t.col0,
                     &t.ncols, &t.max_iter, &t.precision, &t.sampling};
    for (auto* p : f)
      *p = in.u32();
    t.out_offset = in.u64();
  }
  in.expect_done();
  return std::any{std::move(x)};
}

}  // namespace codec

/// Registers the buffer types (idempotent). Call before concurrent use of
/// the registry (type_registry.hpp:60-62); spawn_gpu calls it.
inline void register_types(cafx::type_registry& reg = cafx::type_registry::global()) {
  if (reg.id_of<f32vec>() == cafx::invalid_type_id)
    reg.add<f32vec>("cafxg.f32vec", codec::enc_f32vec, codec::dec_f32vec);
  if (reg.id_of<u32vec>() == cafx::invalid_type_id)
    reg.add<u32vec>("cafxg.u32vec", codec::enc_u32vec, codec::dec_u32vec);
  if (reg.id_of<mandel_tiles>() == cafx::invalid_type_id)
    reg.add<mandel_tiles>("cafxg.mandel_tiles", codec::enc_tiles, codec::dec_tiles);
}

/// A cafx actor whose behaviour is one sm_100a kernel.
class gpu_actor final : public cafx::abstract_actor {
 public:
  gpu_actor(cafx::actor_system& sys, cafxg_ctx* ctx, cafxg_actor* backend, std::string kernel)
      : cafx::abstract_actor(&sys, cafx::actor_addr{sys.node(), sys.next_actor_id()}),
        ctx_(ctx),
        backend_(backend),
        kernel_(std::move(kernel)) {}

  ~gpu_actor() override {
    cafxg_actor_release(backend_);
    // replies whose drain job never ran (the scheduler stopped first)
    for (reply_node* n = replies_.exchange(nullptr); n;) {
      reply_node* next = n->next;
      delete n;
      n = next;
    }
  }

  void enqueue(std::unique_ptr<cafx::envelope> env) override {
    if (env->cat == cafx::envelope::category::exit_signal) {
      on_exit(*env);
      return;
    }
    if (terminated()) {
      fail(*env, cafx::errc::request_down, "compute actor terminated");
      return;
    }
    auto job = std::make_unique<job_t>();
    job->self = cafx::intrusive_ptr<gpu_actor>{this};
    const cafx::message& msg = env->content;
    const void* in[2] = {nullptr, nullptr};
    size_t in_bytes[2] = {0, 0};
    size_t n_in = 0;
    try {
      if (kernel_ == "mandelbrot") {
        if (msg.size() != 1)
          return fail(*env, cafx::errc::interface_mismatch, "expected (mandel_tiles)");
        const auto& t = msg.get<mandel_tiles>(0);
        in[0] = t.tiles.data();
        in_bytes[0] = t.tiles.size() * sizeof(cafxg_mandel_desc);
        n_in = 1;
      } else {
        if (msg.size() != 2)
          return fail(*env, cafx::errc::interface_mismatch, "expected (f32vec, f32vec)");
        const auto& a = msg.get<f32vec>(0);
        const auto& b = msg.get<f32vec>(1);
        in[0] = a.data();
        in[1] = b.data();
        in_bytes[0] = a.size() * sizeof(float);
        in_bytes[1] = b.size() * sizeof(float);
        n_in = 2;
      }
    } catch (const cafx::failure& f) {
      return fail(*env, f.code(), f.what());
    }
    size_t reply = cafxg_actor_reply_bytes(backend_, in, in_bytes, n_in);
    if (reply == 0)
      return fail(*env, static_cast<cafx::errc>(CAFXG_E_TYPE_MISMATCH), cafxg_last_error());
    // the reply vector lives in the context's pinned pool: the device writes
    // into it directly and it moves into the reply message unchanged
    void* out;
    try {
      if (kernel_ == "mandelbrot") {
        job->counts = u32vec(host_allocator<uint32_t>{ctx_});
        job->counts.resize(reply / sizeof(uint32_t));
        out = job->counts.data();
      } else {
        job->floats = f32vec(host_allocator<float>{ctx_});
        job->floats.resize(reply / sizeof(float));
        out = job->floats.data();
      }
    } catch (const std::bad_alloc&) {
      return fail(*env, cafx::errc::config_error, "pinned reply allocation failed");
    }
    job->env = std::move(env);  // keeps the request payload alive
    int s = cafxg_actor_enqueue(backend_, in, in_bytes, n_in, out, reply, &gpu_actor::on_done,
                                job.get());
    if (s != CAFXG_OK)
      return fail(*job->env, static_cast<cafx::errc>(s), cafxg_last_error());
    job.release();  // owned by the backend until on_done
  }

  const std::string& kernel() const noexcept { return kernel_; }

 private:
  struct job_t {
    cafx::intrusive_ptr<gpu_actor> self;
    std::unique_ptr<cafx::envelope> env;
    u32vec counts;
    f32vec floats;
  };

  // Runs on libcafxg's completion thread: the reply goes out through the
  // relay (a scheduler job delivers it from a worker thread).
  static void on_done(void* user, int status) {
    std::unique_ptr<job_t> job{static_cast<job_t*>(user)};
    gpu_actor* self = job->self.get();
    if (self->terminated())
      return;  // pending requesters already got request_down from finalize
    if (status != CAFXG_OK) {
      self->respond(*job->env,
                    cafx::make_message(cafx::error{static_cast<cafx::errc>(status),
                                                   cafxg_last_error()}),
                    true);
      return;
    }
    cafx::message reply = self->kernel_ == "mandelbrot"
                              ? cafx::make_message(std::move(job->counts))
                              : cafx::make_message(std::move(job->floats));
    self->respond(*job->env, std::move(reply), true);
  }

  // local_actor::respond (local_actor.cpp:319-329); `relay`: hand the
  // envelope to the relay instead of delivering on this thread
  void respond(const cafx::envelope& req, cafx::message reply, bool relay = false) {
    std::unique_ptr<cafx::envelope> out;
    if (req.is_request()) {
      auto rid = cafx::envelope::response_id(req.mid);
      drop_pending_request(rid);
      out = cafx::make_envelope(std::move(reply), address(), rid);
    } else if (req.sender) {
      out = cafx::make_envelope(std::move(reply), address());
    } else {
      return;
    }
    if (relay)
      post_reply(req.sender, std::move(out));
    else
      home_system().deliver(req.sender, std::move(out));
  }

  // ---- reply relay --------------------------------------------------------
  struct reply_node {
    cafx::actor_addr to;
    std::unique_ptr<cafx::envelope> env;
    reply_node* next = nullptr;
  };

  // A scheduler job that drains the actor's reply queue on a worker thread.
  // Several may run at once (one is scheduled per empty -> non-empty
  // transition); each reply is taken by exactly one drain (atomic exchange).
  class relay_job final : public cafx::resumable {
   public:
    explicit relay_job(cafx::intrusive_ptr<gpu_actor> a) : actor_(std::move(a)) {}
    resume_result resume(size_t) override {
      actor_->drain_replies();
      return resume_result::finished;
    }
    void ref_job() noexcept override { rc_.fetch_add(1, std::memory_order_relaxed); }
    void deref_job() noexcept override {
      if (rc_.fetch_sub(1, std::memory_order_acq_rel) == 1)
        delete this;
    }

   private:
    cafx::intrusive_ptr<gpu_actor> actor_;
    std::atomic<int> rc_{0};
  };

  void post_reply(const cafx::actor_addr& to, std::unique_ptr<cafx::envelope> env) {
    auto* n = new reply_node{to, std::move(env), nullptr};
    reply_node* head = replies_.load(std::memory_order_relaxed);
    do {
      n->next = head;
    } while (!replies_.compare_exchange_weak(head, n, std::memory_order_release,
                                             std::memory_order_relaxed));
    if (head == nullptr)  // empty -> non-empty: one drain job
      home_system().schedule_job(new relay_job(cafx::intrusive_ptr<gpu_actor>{this}));
  }

  void drain_replies() {
    auto& sys = home_system();
    for (;;) {
      reply_node* h = replies_.exchange(nullptr, std::memory_order_acq_rel);
      if (!h)
        return;
      reply_node* fifo = nullptr;  // the stack holds the newest first
      while (h) {
        reply_node* n = h->next;
        h->next = fifo;
        fifo = h;
        h = n;
      }
      while (fifo) {
        reply_node* n = fifo->next;
        sys.deliver(fifo->to, std::move(fifo->env));
        delete fifo;
        fifo = n;
      }
    }
  }

  void fail(const cafx::envelope& req, cafx::errc code, const std::string& what) {
    respond(req, cafx::make_message(cafx::error{code, what}));
  }

  void on_exit(const cafx::envelope& env) {
    cafx::exit_reason reason = cafx::exit_reason::unhandled_error();
    if (env.content.size() == 3)
      reason = env.content.get<cafx::exit_reason>(2);
    if (!env.hard_kill && reason.is_normal())
      return;  // normal exits do not terminate an actor that is not linked-dead
    bool expected = false;
    if (!quitting_.compare_exchange_strong(expected, true))
      return;
    cafxg_actor_quit(backend_);  // queued requests complete with request_down
    finalize(reason);
    home_system().unregister_actor(address().id);
  }

  cafxg_ctx* ctx_;
  cafxg_actor* backend_;
  std::string kernel_;
  std::atomic<bool> quitting_{false};
  std::atomic<reply_node*> replies_{nullptr};
};

/// spawn_cl for sm_100a: `kernel` names a precompiled kernel of libcafxg
/// ("mandelbrot", "matrix_multiply"); `dims` are the spawn_cl dimensions.
/// Throws cafx::failure (spawn_error, unknown_type, interface_mismatch).
inline cafx::actor spawn_gpu(cafx::actor_system& sys, cafxg_ctx* ctx,
                             const std::string& kernel,
                             std::initializer_list<uint64_t> dims) {
  register_types();
  std::vector<uint64_t> d(dims);
  cafxg_actor* h = nullptr;
  int s = cafxg_spawn(ctx, kernel.c_str(), d.data(), d.size(), &h);
  if (s != CAFXG_OK)
    throw cafx::failure{static_cast<cafx::errc>(s), cafxg_last_error()};
  auto ptr = cafx::make_counted<gpu_actor>(sys, ctx, h, kernel);
  sys.register_actor(cafx::abstract_actor_ptr{ptr.get()});
  return cafx::actor{cafx::abstract_actor_ptr{ptr.get()}};
}

/// Typed variant: one rule (inputs) -> (output), checked by typed sends
/// before the envelope reaches the actor (actor_system.cpp:85-91).
inline cafx::typed_actor spawn_gpu_typed(cafx::actor_system& sys, cafxg_ctx* ctx,
                                         const std::string& kernel,
                                         std::initializer_list<uint64_t> dims) {
  auto h = spawn_gpu(sys, ctx, kernel, dims);
  auto& reg = cafx::type_registry::global();
  cafx::rule r;
  if (kernel == "mandelbrot") {
    r.inputs = {cafx::type_spec::of(reg.id_of<mandel_tiles>())};
    r.outputs = {cafx::type_spec::of(reg.id_of<u32vec>())};
  } else {
    r.inputs = {cafx::type_spec::of(reg.id_of<f32vec>()),
                cafx::type_spec::of(reg.id_of<f32vec>())};
    r.outputs = {cafx::type_spec::of(reg.id_of<f32vec>())};
  }
  return cafx::typed_actor{cafx::abstract_actor_ptr{h.ptr()},
                           cafx::messaging_interface{r}};
}

}  // namespace cafxg
