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
// and the spawn_cl surface itself:
//   auto mm = cafxg::spawn_cl<float*(float*, float*)>(sys, ctx, "matrix_multiply",
//                                                     {size, size});
//   //    typed handle (f32vec, f32vec) -> (f32vec); the template signature is
//   //    checked against the kernel's (cafxg_kernel_signature)
//   cafxg::spawn_cl<uint32_t*(cafxg_mandel_desc*)>(sys, ctx, "mandelbrot", {},
//                                                  cafxg::tuning().block_steps(40));
//   //    tuning overload: launch-shape hints for every request
//   cafxg::spawn_cl<uint32_t*(cafxg_mandel_desc*)>(sys, ctx, "mandelbrot", {},
//       cafx::behavior{[](uint32_t size, uint32_t it) { return mandel_tiles{...}; }},
//       cafx::behavior{[](const u32vec& counts) { return checksum(counts); }});
//   //    data-transformation overload: the actor's interface is
//   //    (uint32, uint32) -> (uint64), the kernel signature stays hidden
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
//    ~actor_system does not wait forever (actor_system.cpp:21-30); a sticky
//    device error (cafxg_ctx_status) terminates the actor the same way, with
//    exit_reason::unhandled_error;
//  * buffer types are registered with wire codecs (type_registry.hpp:74-80),
//    so middleman::publish can serve a GPU actor to remote nodes;
//  * reply relay: the replies of a batch (cafxg_completion_batch() > 1)
//    leave libcafxg's completion thread through a lock-free per-actor queue
//    drained by a job on the cafx scheduler (actor_system::schedule_job,
//    scheduler.hpp:266-274), so the requesters are made runnable from a
//    worker thread (its own deque) and a whole batch of replies costs one
//    external enqueue instead of one each; a lone reply is delivered at once. External
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
#include "cafx/behavior.hpp"
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

/// A cafx actor whose behaviour is one sm_100a kernel, optionally behind a
/// data transformation (spawn_cl's transformation overload): `map_args`
/// turns a request into the kernel's input message, `map_result` turns the
/// kernel's output into the reply. Both are ordinary cafx behaviors, so the
/// transformation is written in the reference's own pattern DSL and its
/// interface derived from it (derive_interface, behavior.hpp:528-532).
class gpu_actor final : public cafx::abstract_actor {
 public:
  gpu_actor(cafx::actor_system& sys, cafxg_ctx* ctx, cafxg_actor* backend, std::string kernel,
            cafx::behavior map_args = {}, cafx::behavior map_result = {})
      : cafx::abstract_actor(&sys, cafx::actor_addr{sys.node(), sys.next_actor_id()}),
        ctx_(ctx),
        backend_(backend),
        kernel_(std::move(kernel)),
        map_args_(std::move(map_args)),
        map_result_(std::move(map_result)) {}

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
    // the kernel's input message: the request itself, or what map_args makes
    // of it (kept in the job: the buffers handed to the backend live in it)
    job->input = env->content;
    if (map_args_.defined()) {
      cafx::message req = env->content;
      cafx::match_outcome out;
      try {
        out = cafx::match(map_args_, req);
      } catch (const cafx::failure& f) {
        return fail(*env, f.code(), f.what());
      }
      if (!out.matched || !out.response)
        return fail(*env, cafx::errc::type_mismatch,
                    "request matches no case of the compute actor's data transformation");
      job->input = std::move(*out.response);
    }
    const cafx::message& msg = job->input;
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
    if (s != CAFXG_OK) {
      fail(*job->env, static_cast<cafx::errc>(s), cafxg_last_error());
      // the context was lost through another actor's request: terminate too
      if (s == CAFXG_E_DOWN && cafxg_ctx_status(ctx_) != CAFXG_OK)
        terminate(cafx::exit_reason::unhandled_error());
      return;
    }
    job.release();  // owned by the backend until on_done
  }

  const std::string& kernel() const noexcept { return kernel_; }

 private:
  struct job_t {
    cafx::intrusive_ptr<gpu_actor> self;
    std::unique_ptr<cafx::envelope> env;
    cafx::message input;
    u32vec counts;
    f32vec floats;
  };

  // Runs on libcafxg's completion thread: the reply goes out through the
  // relay (a scheduler job delivers it -- and applies map_result -- on a
  // worker thread).
  static void on_done(void* user, int status) {
    std::unique_ptr<job_t> job{static_cast<job_t*>(user)};
    gpu_actor* self = job->self.get();
    if (self->terminated())
      return;  // pending requesters already got request_down from finalize
    if (status != CAFXG_OK) {
      // (delivered here, not through the relay: a terminating actor's
      // requester gets the error before monitors get the down message)
      self->respond(*job->env,
                    cafx::make_message(cafx::error{static_cast<cafx::errc>(status),
                                                   cafxg_last_error()}));
      // a sticky device error: the backend cannot serve anything any more,
      // so the actor terminates (monitors, links and pending requesters fire,
      // abstract_actor.cpp:108-134) instead of failing requests one by one
      if (cafxg_ctx_status(self->ctx_) != CAFXG_OK)
        self->terminate(cafx::exit_reason::unhandled_error());
      return;
    }
    cafx::message reply = self->kernel_ == "mandelbrot"
                              ? cafx::make_message(std::move(job->counts))
                              : cafx::make_message(std::move(job->floats));
    // replies of a batch go through the relay (one external enqueue for all
    // of them); a lone reply is delivered right here -- through the relay it
    // would wait for an idle cafx worker to wake (up to the 1 ms steal
    // back-off) for no saving. map_result always runs on a worker.
    const bool relay = self->map_result_.defined() || cafxg_completion_batch() > 1;
    self->respond(*job->env, std::move(reply), relay, self->map_result_.defined());
  }

  // local_actor::respond (local_actor.cpp:319-329). `relay`: hand the reply
  // to the relay instead of delivering on this thread; `post`: the relay
  // passes it through map_result first.
  void respond(const cafx::envelope& req, cafx::message reply, bool relay = false,
               bool post = false) {
    uint64_t rid = 0;
    if (req.is_request()) {
      rid = cafx::envelope::response_id(req.mid);
      drop_pending_request(rid);
    } else if (!req.sender) {
      return;
    }
    if (relay) {
      post_reply(new reply_node{req.sender, rid, std::move(reply), post, nullptr});
      return;
    }
    home_system().deliver(req.sender, rid ? cafx::make_envelope(std::move(reply), address(), rid)
                                          : cafx::make_envelope(std::move(reply), address()));
  }

  void fail(const cafx::envelope& req, cafx::errc code, const std::string& what) {
    respond(req, cafx::make_message(cafx::error{code, what}));
  }

  // ---- reply relay --------------------------------------------------------
  struct reply_node {
    cafx::actor_addr to;
    uint64_t rid;          // response id, 0 for an async reply
    cafx::message msg;
    bool post;             // apply map_result before delivery
    reply_node* next;
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

  void post_reply(reply_node* n) {
    reply_node* head = replies_.load(std::memory_order_relaxed);
    do {
      n->next = head;
    } while (!replies_.compare_exchange_weak(head, n, std::memory_order_release,
                                             std::memory_order_relaxed));
    if (head == nullptr)  // empty -> non-empty: one drain job
      home_system().schedule_job(new relay_job(cafx::intrusive_ptr<gpu_actor>{this}));
  }

  // map_result of a kernel reply; a reply it does not match becomes an error
  cafx::message transform_result(cafx::message m) {
    try {
      auto out = cafx::match(map_result_, m);
      if (out.matched && out.response)
        return std::move(*out.response);
      return cafx::make_message(cafx::error{cafx::errc::type_mismatch,
                                            "kernel result matches no case of map_result"});
    } catch (const cafx::failure& f) {
      return cafx::make_message(cafx::error{f.code(), f.what()});
    }
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
        cafx::message m = fifo->post ? transform_result(std::move(fifo->msg))
                                     : std::move(fifo->msg);
        sys.deliver(fifo->to, fifo->rid ? cafx::make_envelope(std::move(m), address(), fifo->rid)
                                        : cafx::make_envelope(std::move(m), address()));
        delete fifo;
        fifo = n;
      }
    }
  }

  void on_exit(const cafx::envelope& env) {
    cafx::exit_reason reason = cafx::exit_reason::unhandled_error();
    if (env.content.size() == 3)
      reason = env.content.get<cafx::exit_reason>(2);
    if (!env.hard_kill && reason.is_normal())
      return;  // normal exits do not terminate an actor that is not linked-dead
    terminate(reason);
  }

  void terminate(const cafx::exit_reason& reason) {
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
  cafx::behavior map_args_, map_result_;
  std::atomic<bool> quitting_{false};
  std::atomic<reply_node*> replies_{nullptr};
};

// ---- spawn_cl ----------------------------------------------------------------

/// Element type of a kernel buffer parameter -> the message payload type that
/// carries it and its token in the normalised signature text.
template <class T>
struct buffer_traits;
template <>
struct buffer_traits<float> {
  using type = f32vec;
  static constexpr const char* token = "f32*";
};
template <>
struct buffer_traits<uint32_t> {
  using type = u32vec;
  static constexpr const char* token = "u32*";
};
template <>
struct buffer_traits<cafxg_mandel_desc> {
  using type = mandel_tiles;
  static constexpr const char* token = "mandel_desc*";
};

/// spawn_cl's template argument `Out*(In*...)`: the
/// kernel signature normalised to a result type instead of the trailing
/// output parameter.
template <class Sig>
struct kernel_sig;
template <class R, class... Ts>
struct kernel_sig<R*(Ts*...)> {
  static std::string text() {
    std::string s = std::string(buffer_traits<std::remove_cv_t<R>>::token) + "(";
    bool first = true;
    ((s += (first ? "" : ","), s += buffer_traits<std::remove_cv_t<Ts>>::token, first = false),
     ...);
    return s + ")";
  }
  // the typed rule (In buffers...) -> (Out buffer)
  static cafx::rule rule(const cafx::type_registry& reg) {
    cafx::rule r;
    r.inputs = {cafx::type_spec::of(reg.id_of<typename buffer_traits<std::remove_cv_t<Ts>>::type>())...};
    r.outputs = {cafx::type_spec::of(reg.id_of<typename buffer_traits<std::remove_cv_t<R>>::type>())};
    return r;
  }
  // payload types of the kernel input message / of the kernel output
  static std::vector<cafx::type_spec> input_specs(const cafx::type_registry& reg) {
    return rule(reg).inputs;
  }
};

namespace detail {

inline cafxg_actor* spawn_backend(cafxg_ctx* ctx, const std::string& kernel, const char* sig,
                                  std::initializer_list<uint64_t> dims,
                                  const cafxg_tuning* tuning) {
  register_types();
  std::vector<uint64_t> d(dims);
  cafxg_actor* h = nullptr;
  int s = cafxg_spawn_ex(ctx, kernel.c_str(), sig, d.data(), d.size(), tuning, &h);
  if (s != CAFXG_OK)
    throw cafx::failure{static_cast<cafx::errc>(s), cafxg_last_error()};
  return h;
}

inline cafx::actor make_handle(cafx::actor_system& sys, cafxg_ctx* ctx, cafxg_actor* h,
                               const std::string& kernel, cafx::behavior map_args = {},
                               cafx::behavior map_result = {}) {
  auto ptr = cafx::make_counted<gpu_actor>(sys, ctx, h, kernel, std::move(map_args),
                                           std::move(map_result));
  sys.register_actor(cafx::abstract_actor_ptr{ptr.get()});
  return cafx::actor{cafx::abstract_actor_ptr{ptr.get()}};
}

}  // namespace detail

/// spawn_cl for sm_100a: `kernel` names a precompiled kernel of libcafxg
/// ("mandelbrot", "matrix_multiply"); `dims` are the spawn_cl dimensions.
/// Throws cafx::failure (spawn_error, unknown_type, interface_mismatch).
inline cafx::actor spawn_gpu(cafx::actor_system& sys, cafxg_ctx* ctx,
                             const std::string& kernel,
                             std::initializer_list<uint64_t> dims) {
  cafxg_actor* h = detail::spawn_backend(ctx, kernel, nullptr, dims, nullptr);
  return detail::make_handle(sys, ctx, h, kernel);
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

/// spawn_cl's tuning overload: launch-shape hints for every request of the
/// actor (include/cafxg.h, cafxg_tuning). Zero fields keep the defaults.
struct tuning : cafxg_tuning {
  tuning() : cafxg_tuning{} {}
  tuning& block_steps(uint32_t v) { cafxg_tuning::block_steps = v; return *this; }
  tuning& max_ctas(uint32_t v) { cafxg_tuning::max_ctas = v; return *this; }
  tuning& sgemm_mode(uint32_t v) { cafxg_tuning::sgemm_mode = v; return *this; }
  tuning& sgemm_splits(uint32_t v) { cafxg_tuning::sgemm_splits = v; return *this; }
};

/// spawn_cl<Out*(In*...)>(sys, ctx, kernel, dims[, tuning]) -- PAPER.md:
/// 357-361 with the OpenCL source replaced by a precompiled sm_100a kernel.
/// The template signature is checked against the kernel's registered one
/// (cafxg_kernel_signature) before anything is spawned: a mismatch throws
/// failure{interface_mismatch}. Returns a typed handle whose one rule is
/// (In buffers...) -> (Out buffer), e.g. spawn_cl<float*(float*, float*)>
/// -> (f32vec, f32vec) -> (f32vec).
template <class Sig>
cafx::typed_actor spawn_cl(cafx::actor_system& sys, cafxg_ctx* ctx, const std::string& kernel,
                           std::initializer_list<uint64_t> dims, const tuning& t = tuning{}) {
  register_types();
  const std::string sig = kernel_sig<Sig>::text();
  cafxg_actor* h = detail::spawn_backend(ctx, kernel, sig.c_str(), dims, &t);
  auto a = detail::make_handle(sys, ctx, h, kernel);
  return cafx::typed_actor{cafx::abstract_actor_ptr{a.ptr()},
                           cafx::messaging_interface{
                               kernel_sig<Sig>::rule(cafx::type_registry::global())}};
}

/// spawn_cl's data-transformation overload: the actor shows other actors an
/// interface of its own instead of the kernel signature. map_args runs on the
/// sender's thread (inside enqueue), map_result on a cafx worker (the reply
/// relay), both possibly concurrently for different requests: they must not
/// share unsynchronised state (stateless lambdas, as in the examples).
/// `map_args` maps a
/// request to the kernel's input message (each of its cases must produce
/// exactly Sig's input buffers), `map_result` maps the kernel's output buffer
/// to the reply (its one case takes Sig's output buffer). The typed handle's
/// rules are map_args' inputs -> map_result's outputs; a request matching no
/// case of map_args is answered with error{type_mismatch}. Both behaviors
/// must be typable (no catch-all), else failure{interface_mismatch}.
template <class Sig>
cafx::typed_actor spawn_cl(cafx::actor_system& sys, cafxg_ctx* ctx, const std::string& kernel,
                           std::initializer_list<uint64_t> dims, cafx::behavior map_args,
                           cafx::behavior map_result, const tuning& t = tuning{}) {
  register_types();
  auto& reg = cafx::type_registry::global();
  const cafx::rule krule = kernel_sig<Sig>::rule(reg);
  auto in_if = cafx::derive_interface(map_args);
  auto out_if = cafx::derive_interface(map_result);
  if (!in_if || !out_if || in_if->empty() || out_if->size() != 1)
    throw cafx::failure{cafx::errc::interface_mismatch,
                        "spawn_cl: map_args / map_result must be typable behaviors "
                        "(map_result with exactly one case)"};
  const cafx::rule& post = out_if->rules().front();
  if (post.inputs != krule.outputs)
    throw cafx::failure{cafx::errc::interface_mismatch,
                        "spawn_cl: map_result must take the kernel's output " +
                            kernel_sig<Sig>::text()};
  std::vector<cafx::rule> rules;
  for (const cafx::rule& pre : in_if->rules()) {
    if (pre.outputs != krule.inputs)
      throw cafx::failure{cafx::errc::interface_mismatch,
                          "spawn_cl: every map_args case must produce the kernel's inputs " +
                              kernel_sig<Sig>::text() + ", got " + cafx::to_string(pre)};
    cafx::rule r;
    r.inputs = pre.inputs;
    r.outputs = post.outputs;
    rules.push_back(std::move(r));
  }
  const std::string sig = kernel_sig<Sig>::text();
  cafxg_actor* h = detail::spawn_backend(ctx, kernel, sig.c_str(), dims, &t);
  auto a = detail::make_handle(sys, ctx, h, kernel, std::move(map_args), std::move(map_result));
  return cafx::typed_actor{cafx::abstract_actor_ptr{a.ptr()},
                           cafx::messaging_interface{std::move(rules)}};
}

}  // namespace cafxg
