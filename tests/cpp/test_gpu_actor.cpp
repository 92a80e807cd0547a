// GPU test of the drop-in on the UNMODIFIED reference runtime: cafx actors
// (scoped, event-based, typed handles) talk to include/cafxg/gpu_actor.hpp
// compute actors exactly as they would to CAF's OpenCL actors. Links the
// reference compiled from its own sources (oracle/_ref/libcafx_ref.so) and
// libcafxg.so. Prints one PASS/FAIL line per check; exit code 0 iff all pass.
// Built by tests/cpp/Makefile, run by tests/test_cafx_adapter_gpu.py.
#include <atomic>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <thread>
#include <variant>
#include <vector>

#include "cafx/actor_system.hpp"
#include "cafx/atoms.hpp"
#include "cafx/bench/bench.hpp"
#include "cafx/detail/fnv.hpp"
#include "cafx/io/middleman.hpp"
#include "cafx/scoped_actor.hpp"
#include "cafxg/gpu_actor.hpp"

using namespace std::chrono_literals;

static int failures = 0;
static cafxg_ctx* lost_ctx = nullptr;  // section 9's context (closed last)

static void check(bool ok, const std::string& name) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", name.c_str());
  std::fflush(stdout);
  if (!ok)
    ++failures;
}

static cafxg_mandel_desc ref_desc(uint32_t size, uint32_t it) {
  cafxg_mandel_desc d{};
  d.x0 = -1.5; d.x1 = 0.5; d.y0 = -1.0; d.y1 = 1.0;
  d.width = d.height = size;
  d.nrows = d.ncols = size;
  d.max_iter = it;
  d.precision = CAFXG_FP64;
  d.sampling = CAFXG_CORNER;
  return d;
}

static cafxg_mandel_desc storm_tile(std::mt19937_64& rng) {
  cafxg_mandel_desc d{};
  uint64_t kx = rng() % (3 * 512 - 64 + 1), ky = rng() % (2 * 512 - 64 + 1);
  d.x0 = -2.0 + kx / 512.0; d.x1 = d.x0 + 0.125;
  d.y0 = -1.0 + ky / 512.0; d.y1 = d.y0 + 0.125;
  d.width = d.height = d.nrows = d.ncols = 64;
  d.max_iter = 256;
  d.precision = CAFXG_FP64;
  d.sampling = CAFXG_CENTRE;
  return d;
}

// expected counts of a storm tile through the reference's own cell
// (bench.cpp:367) and the generalised coordinate contract (cafxg.h)
static cafxg::u32vec expect_tile(const cafxg_mandel_desc& d) {
  cafxg::u32vec out(64 * 64);
  for (uint32_t r = 0; r < 64; ++r) {
    volatile double ky = r + 0.5;
    volatile double qi = ky * (d.y1 - d.y0);
    double ci = d.y0 + qi / 64.0;
    for (uint32_t c = 0; c < 64; ++c) {
      volatile double kx = c + 0.5;
      volatile double qr = kx * (d.x1 - d.x0);
      double cr = d.x0 + qr / 64.0;
      out[r * 64 + c] = cafx::bench::mandelbrot_cell(cr, ci, 256);
    }
  }
  return out;
}

int main() {
  cafxg_ctx* ctx = nullptr;
  if (cafxg_open(1, &ctx) != CAFXG_OK) {
    std::printf("FAIL cafxg_open: %s\n", cafxg_last_error());
    return 1;
  }
  {
    cafx::actor_system sys;
    cafx::scoped_actor self{sys};

    // 1. run_mandelbrot(256, 100)'s image through a request, checksum
    //    bit-exact (bench.cpp:481-505; golden 12958954340663424292)
    auto mb = cafxg::spawn_gpu(sys, ctx, "mandelbrot", {});
    {
      cafxg::mandel_tiles req{{ref_desc(256, 100)}};
      auto res = self->request(mb, cafx::make_message(req), 60s);
      bool ok = std::holds_alternative<cafx::message>(res);
      if (ok) {
        const auto& counts = std::get<cafx::message>(res).get<cafxg::u32vec>(0);
        uint64_t h = cafx::detail::fnv1a_seed;
        for (uint32_t c : counts)
          h = cafx::detail::fnv1a_u32(h, c);
        ok = counts.size() == 256 * 256 && h == 12958954340663424292ull;
      }
      check(ok, "request run_mandelbrot(256,100) image -> checksum golden");
    }

    // 2. matrix_multiply: spawn_cl<float*(float*,float*)>(.., {size, size})
    {
      const uint32_t n = 128;
      auto mm = cafxg::spawn_gpu(sys, ctx, "matrix_multiply", {n, n});
      cafxg::f32vec a(n * n), b(n * n);
      std::mt19937_64 rng(5);
      std::uniform_real_distribution<float> u(-1.0f, 1.0f);
      for (auto& x : a) x = u(rng);
      for (auto& x : b) x = u(rng);
      auto res = self->request(mm, cafx::make_message(a, b), 60s);
      bool ok = std::holds_alternative<cafx::message>(res);
      double worst = 0;
      if (ok) {
        const auto& c = std::get<cafx::message>(res).get<cafxg::f32vec>(0);
        ok = c.size() == n * n;
        for (uint32_t i = 0; ok && i < n; i += 7) {
          double num = 0, den = 0;
          for (uint32_t j = 0; j < n; ++j) {
            double r = 0;
            for (uint32_t k = 0; k < n; ++k)
              r += (double)a[i * n + k] * (double)b[k * n + j];
            num = std::max(num, std::fabs(c[i * n + j] - r));
            den = std::max(den, std::fabs(r));
          }
          worst = std::max(worst, num / den);
        }
        ok = ok && worst <= 1e-5;
      }
      check(ok, "matrix_multiply actor reply within 1e-5 (err " + std::to_string(worst) + ")");

      // wrong arity -> error reply, the requester's failure path
      auto bad = self->request(mm, cafx::make_message(a), 30s);
      check(std::holds_alternative<cafx::error>(bad) &&
                std::get<cafx::error>(bad).code == cafx::errc::interface_mismatch,
            "wrong arity -> error(interface_mismatch) reply");
      auto bad2 = self->request(mm, cafx::make_message(a, cafxg::f32vec(3)), 30s);
      check(std::holds_alternative<cafx::error>(bad2) &&
                std::get<cafx::error>(bad2).code == cafx::errc::type_mismatch,
            "wrong buffer size -> error(type_mismatch) reply");
    }

    // 3. 64 event-based client actors, each a chain of 40 sync_send(...)
    //    .then(...) storm tiles (one outstanding request per client,
    //    local_actor.cpp:99-101); every reply checked against the reference's
    //    own mandelbrot_cell.
    {
      const int clients = 64, per = 40;
      std::atomic<int> good{0}, bad{0}, finished{0};
      for (int c = 0; c < clients; ++c) {
        auto client = sys.spawn([&, c, mb](cafx::event_based_actor* me) {
          auto rng = std::make_shared<std::mt19937_64>(1000 + c);
          // each `go` issues the next sync request; its response handler
          // re-sends `go` to self until `per` requests are done
          return cafx::behavior{
              [=, &good, &bad, &finished](uint32_t k) {
                auto d = storm_tile(*rng);
                cafx::actor self_handle{cafx::abstract_actor_ptr{me}};
                me->sync_send(mb, cafx::make_message(cafxg::mandel_tiles{{d}}))
                    .then(
                        [=, &good, &bad, &finished](const cafxg::u32vec& counts) {
                          (counts == expect_tile(d) ? good : bad)++;
                          if (k + 1 < (uint32_t)per) {
                            me->send(self_handle, cafx::make_message(k + 1));
                          } else {
                            finished++;
                            me->quit();
                          }
                        },
                        [=, &bad, &finished](const cafx::error&) {
                          bad++;
                          finished++;
                          me->quit();
                        });
              },
          };
        });
        sys.anon_send(client, cafx::make_message(uint32_t{0}));
      }
      auto t0 = std::chrono::steady_clock::now();
      while (finished.load() < clients &&
             std::chrono::steady_clock::now() - t0 < 120s)
        std::this_thread::sleep_for(5ms);
      check(finished.load() == clients && good.load() == clients * per && bad.load() == 0,
            "64 event-based clients x 40 sync_send storm tiles, all replies exact (" +
                std::to_string(good.load()) + " good, " + std::to_string(bad.load()) + " bad)");
    }

    // 4. async send with a sender: reply delivered to the sender's mailbox
    {
      cafx::scoped_actor other{sys};
      std::mt19937_64 rng(77);
      auto d = storm_tile(rng);
      other->send(mb, cafx::make_message(cafxg::mandel_tiles{{d}}));
      bool got = false;
      other->receive(cafx::behavior{[&](const cafxg::u32vec& counts) {
                       got = counts == expect_tile(d);
                     }},
                     60s);
      check(got, "async send -> reply to the sender (local_actor.cpp:325-327)");
    }

    // 5. typed handle: the interface check rejects a mistyped send before
    //    it reaches the actor (actor_system.cpp:85-91)
    {
      auto typed = cafxg::spawn_gpu_typed(sys, ctx, "mandelbrot", {});
      bool threw = false;
      try {
        sys.anon_send(typed, cafx::make_message(uint32_t{7}));
      } catch (const cafx::failure& f) {
        threw = f.code() == cafx::errc::type_mismatch;
      }
      check(threw, "typed gpu actor: mistyped send throws type_mismatch (actor_system.cpp:85-91)");
      std::mt19937_64 rng(78);
      auto d = storm_tile(rng);
      auto res = self->request(typed, cafx::make_message(cafxg::mandel_tiles{{d}}), 60s);
      check(std::holds_alternative<cafx::message>(res) &&
                std::get<cafx::message>(res).get<cafxg::u32vec>(0) == expect_tile(d),
            "typed gpu actor request");
    }

    // 6. wire codec round trip (what middleman::publish would send)
    {
      std::mt19937_64 rng(79);
      cafxg::mandel_tiles t{{storm_tile(rng), storm_tile(rng)}};
      auto msg = cafx::make_message(t, cafxg::u32vec{1, 2, 0xfffffffeu},
                                    cafxg::f32vec{1.5f, -0.0f});
      auto back = cafx::deserialize(cafx::serialize(msg));
      check(back == msg, "buffer types serialize/deserialize (BASP payload codecs)");
    }

    // 7. remote compute actors over BASP: a second
    //    actor system reaches published GPU actors through the unmodified
    //    middleman over TCP on 127.0.0.1; requests, replies and error replies
    //    cross the wire through the registered codecs (middleman.cpp:421-447).
    {
      cafx::io::middleman server_mm{sys};
      cafx::actor_system client_sys;
      cafx::io::middleman client_mm{client_sys};
      auto typed = cafxg::spawn_gpu_typed(sys, ctx, "mandelbrot", {});
      auto port = server_mm.publish(typed, 0);
      auto remote = client_mm.remote_actor("127.0.0.1", port, typed.interface());
      cafx::scoped_actor cself{client_sys};
      std::mt19937_64 rng(80);
      const int n_remote = 200;
      int good = 0;
      auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < n_remote; ++i) {
        cafxg::mandel_tiles t{{storm_tile(rng), storm_tile(rng)}};
        auto res = cself->request(remote, cafx::make_message(t), 60s);
        if (!std::holds_alternative<cafx::message>(res))
          continue;
        const auto& counts = std::get<cafx::message>(res).get<cafxg::u32vec>(0);
        auto e0 = expect_tile(t.tiles[0]), e1 = expect_tile(t.tiles[1]);
        e0.insert(e0.end(), e1.begin(), e1.end());
        good += counts == e0;
      }
      double ms = std::chrono::duration<double, std::milli>(
                      std::chrono::steady_clock::now() - t0).count();
      check(good == n_remote, "remote typed gpu actor over TCP: " + std::to_string(good) + "/" +
                                  std::to_string(n_remote) + " two-tile requests exact (" +
                                  std::to_string(ms / n_remote) + " ms/request round trip)");

      const uint32_t n = 256;
      auto mm = cafxg::spawn_gpu(sys, ctx, "matrix_multiply", {n, n});
      auto port2 = server_mm.publish(mm, 0);
      auto rmm = client_mm.remote_actor("127.0.0.1", port2);
      cafxg::f32vec a(n * n), b(n * n);
      std::uniform_real_distribution<float> u(-1.0f, 1.0f);
      for (auto& x : a) x = u(rng);
      for (auto& x : b) x = u(rng);
      auto res = cself->request(rmm, cafx::make_message(a, b), 60s);
      double worst = 1;
      if (std::holds_alternative<cafx::message>(res)) {
        const auto& c = std::get<cafx::message>(res).get<cafxg::f32vec>(0);
        worst = c.size() == n * n ? 0 : 1;
        for (uint32_t i = 0; c.size() == n * n && i < n; i += 11) {
          double num = 0, den = 0;
          for (uint32_t j = 0; j < n; ++j) {
            double r = 0;
            for (uint32_t k = 0; k < n; ++k)
              r += (double)a[i * n + k] * (double)b[k * n + j];
            num = std::max(num, std::fabs(c[i * n + j] - r));
            den = std::max(den, std::fabs(r));
          }
          worst = std::max(worst, num / den);
        }
      }
      check(worst <= 1e-5, "remote matrix_multiply over TCP within 1e-5 (err " +
                               std::to_string(worst) + ")");
      auto bad = cself->request(rmm, cafx::make_message(a), 30s);
      check(std::holds_alternative<cafx::error>(bad) &&
                std::get<cafx::error>(bad).code == cafx::errc::interface_mismatch,
            "remote wrong arity -> error(interface_mismatch) reply over the wire");
    }

    // 8. the spawn_cl surface: signature template checked
    //    against the kernel, tuning overload, data-transformation overload
    {
      // (a) spawn_cl<float*(float*,float*)> -> typed (f32vec, f32vec) -> (f32vec)
      const uint32_t n = 256;
      auto mm = cafxg::spawn_cl<float*(float*, float*)>(sys, ctx, "matrix_multiply", {n, n});
      cafxg::f32vec a(n * n, 0.0f), b(n * n, 0.0f);
      for (uint32_t i = 0; i < n; ++i) {
        a[i * n + i] = 2.0f;           // A = 2 I
        b[i * n + (n - 1 - i)] = 1.0f;  // B = anti-identity
      }
      auto res = self->request(mm, cafx::make_message(a, b), 60s);
      bool ok = std::holds_alternative<cafx::message>(res);
      if (ok) {
        const auto& c = std::get<cafx::message>(res).get<cafxg::f32vec>(0);
        for (uint32_t i = 0; ok && i < n; ++i)
          for (uint32_t j = 0; ok && j < n; ++j)
            ok = c[i * n + j] == (j == n - 1 - i ? 2.0f : 0.0f);
      }
      auto& reg = cafx::type_registry::global();
      cafx::rule want;
      want.inputs = {cafx::type_spec::of(reg.id_of<cafxg::f32vec>()),
                     cafx::type_spec::of(reg.id_of<cafxg::f32vec>())};
      want.outputs = {cafx::type_spec::of(reg.id_of<cafxg::f32vec>())};
      check(ok && mm.interface() == cafx::messaging_interface{want},
            "spawn_cl<float*(float*,float*)>: typed (f32vec,f32vec)->(f32vec), reply exact");
      // typed sends are checked at the sender (actor_system.cpp:85-91)
      bool threw = false;
      try {
        sys.anon_send(mm, cafx::make_message(a));
      } catch (const cafx::failure& f) {
        threw = f.code() == cafx::errc::type_mismatch;
      }
      check(threw, "typed handle from the signature rejects a wrong send at the sender");
    }
    {
      // (b) a signature that does not match the kernel's
      bool threw = false;
      try {
        cafxg::spawn_cl<float*(float*)>(sys, ctx, "matrix_multiply", {64, 64});
      } catch (const cafx::failure& f) {
        threw = f.code() == cafx::errc::interface_mismatch;
      }
      bool threw2 = false;
      try {
        cafxg::spawn_cl<uint32_t*(float*, float*)>(sys, ctx, "matrix_multiply", {64, 64});
      } catch (const cafx::failure& f) {
        threw2 = f.code() == cafx::errc::interface_mismatch;
      }
      check(threw && threw2, "spawn_cl with a mismatched signature -> failure(interface_mismatch)");
    }
    {
      // (c) tuning overload: launch-shape hints; bad values fail the spawn
      auto mb = cafxg::spawn_cl<uint32_t*(cafxg_mandel_desc*)>(
          sys, ctx, "mandelbrot", {}, cafxg::tuning().block_steps(24).max_ctas(64));
      cafxg_mandel_desc d{};
      d.x0 = -0.75; d.x1 = -0.73; d.y0 = 0.10; d.y1 = 0.12;
      d.width = d.height = d.nrows = d.ncols = 192;
      d.max_iter = 1000;
      d.precision = CAFXG_FP64;
      d.sampling = CAFXG_CENTRE;
      auto res = self->request(mb, cafx::make_message(cafxg::mandel_tiles{{d}}), 60s);
      bool ok = std::holds_alternative<cafx::message>(res);
      if (ok) {
        const auto& counts = std::get<cafx::message>(res).get<cafxg::u32vec>(0);
        for (uint32_t r = 0; ok && r < 192; r += 7)
          for (uint32_t c = 0; ok && c < 192; ++c) {
            const double ci = d.y0 + (((double)r + 0.5) * (d.y1 - d.y0)) / 192;
            const double cr = d.x0 + (((double)c + 0.5) * (d.x1 - d.x0)) / 192;
            ok = counts[r * 192 + c] == cafx::bench::mandelbrot_cell(cr, ci, 1000);
          }
      }
      bool threw = false;
      try {
        cafxg::spawn_cl<uint32_t*(cafxg_mandel_desc*)>(sys, ctx, "mandelbrot", {},
                                                       cafxg::tuning().block_steps(20));
      } catch (const cafx::failure& f) {
        threw = f.code() == cafx::errc::config_error;
      }
      check(ok && threw,
            "spawn_cl tuning overload: block_steps 24 / max_ctas 64 exact; block_steps 20 "
            "-> failure(config_error)");
    }
    {
      // (d) data-transformation overload: (uint32 size, uint32 max_iter) ->
      //     run_mandelbrot's image on the GPU -> its collector checksum; the
      //     kernel signature stays hidden behind the actor's own interface
      auto rm = cafxg::spawn_cl<uint32_t*(cafxg_mandel_desc*)>(
          sys, ctx, "mandelbrot", {},
          cafx::behavior{[](uint32_t size, uint32_t it) {
            return cafxg::mandel_tiles{{ref_desc(size, it)}};
          }},
          cafx::behavior{[](const cafxg::u32vec& counts) {
            uint64_t h = cafx::detail::fnv1a_seed;
            for (uint32_t c : counts)
              h = cafx::detail::fnv1a_u32(h, c);
            return h;
          }});
      auto res = self->request(rm, cafx::make_message(uint32_t{256}, uint32_t{100}), 60s);
      bool ok = std::holds_alternative<cafx::message>(res) &&
                std::get<cafx::message>(res).get<uint64_t>(0) == 12958954340663424292ull;
      auto& reg = cafx::type_registry::global();
      ok = ok && rm.interface().size() == 1 &&
           rm.interface().rules()[0].inputs.size() == 2 &&
           rm.interface().rules()[0].outputs ==
               std::vector<cafx::type_spec>{cafx::type_spec::of(reg.id_of<uint64_t>())};
      check(ok, "spawn_cl transformation: (uint32 256, uint32 100) -> checksum golden, "
                "typed (u32,u32)->(u64)");
      // a request the transformation does not match -> error reply
      auto bad = self->request(cafx::actor_cast(rm), cafx::make_message(1.5f), 30s);
      check(std::holds_alternative<cafx::error>(bad) &&
                std::get<cafx::error>(bad).code == cafx::errc::type_mismatch,
            "spawn_cl transformation: unmatched request -> error(type_mismatch)");
      // map_args must produce the kernel's inputs
      bool threw = false;
      try {
        cafxg::spawn_cl<uint32_t*(cafxg_mandel_desc*)>(
            sys, ctx, "mandelbrot", {},
            cafx::behavior{[](uint32_t n) { return cafxg::f32vec(n); }},
            cafx::behavior{[](const cafxg::u32vec& c) { return (uint32_t)c.size(); }});
      } catch (const cafx::failure& f) {
        threw = f.code() == cafx::errc::interface_mismatch;
      }
      check(threw, "spawn_cl transformation whose map_args misses the kernel inputs -> "
                   "failure(interface_mismatch)");
    }

    // 10. a large request (>= 1M pixels leaves the batching path: row bands
    //     over every device of the context -- with CAFXG_VIRTUAL_DEVICES, the
    //     per-device issuer threads -- and overlapped waves into the reply)
    {
      auto big = cafxg::spawn_gpu(sys, ctx, "mandelbrot", {});
      cafxg_mandel_desc d{};
      d.x0 = -2.0; d.x1 = 1.0; d.y0 = -1.0; d.y1 = 1.0;
      d.width = d.ncols = 1536;
      d.height = d.nrows = 1024;
      d.max_iter = 200;
      d.precision = CAFXG_FP64;
      d.sampling = CAFXG_CENTRE;
      auto res = self->request(big, cafx::make_message(cafxg::mandel_tiles{{d}}), 60s);
      bool ok = std::holds_alternative<cafx::message>(res);
      if (ok) {
        const auto& counts = std::get<cafx::message>(res).get<cafxg::u32vec>(0);
        ok = counts.size() == 1536u * 1024u;
        for (uint32_t r = 0; ok && r < 1024; r += 31)
          for (uint32_t c = 0; ok && c < 1536; ++c) {
            const double ci = d.y0 + (((double)r + 0.5) * (d.y1 - d.y0)) / 1024;
            const double cr = d.x0 + (((double)c + 0.5) * (d.x1 - d.x0)) / 1536;
            ok = counts[r * 1536 + c] == cafx::bench::mandelbrot_cell(cr, ci, 200);
          }
      }
      check(ok, "large request (1.5M pixels) through the actor: bands over every device, "
                "sampled rows = the reference's mandelbrot_cell");
    }

    // 9. device loss: a sticky CUDA error (simulated on a second context:
    //    CAFXG_SIMULATE_DEVICE_LOSS makes its 2nd completion report
    //    cudaErrorLaunchFailure, as a real fault would) terminates the compute
    //    actor: the failing request gets an error reply, monitors receive
    //    down(unhandled_error), later requests get request_down
    {
      setenv("CAFXG_SIMULATE_DEVICE_LOSS", "2", 1);
      const int os = cafxg_open(1, &lost_ctx);
      unsetenv("CAFXG_SIMULATE_DEVICE_LOSS");
      check(os == CAFXG_OK, "second context for the device-loss check");
      auto mb = cafxg::spawn_gpu(sys, lost_ctx, "mandelbrot", {});
      cafx::monitor(self.handle(), mb);
      std::mt19937_64 rng(4242);
      auto d = storm_tile(rng);
      auto r1 = self->request(mb, cafx::make_message(cafxg::mandel_tiles{{d}}), 60s);
      auto r2 = self->request(mb, cafx::make_message(cafxg::mandel_tiles{{d}}), 60s);
      bool down = false, unhandled = false;
      int reason_kind = -1;
      const bool got = self->receive(cafx::behavior{[&](cafx::down_atom, cafx::actor_addr src,
                                                        cafx::exit_reason reason) {
                                       down = src == mb.address();
                                       reason_kind = (int)reason.k;
                                       unhandled =
                                           reason.k == cafx::exit_reason::kind::unhandled_error;
                                     }},
                                     30s);
      if (!(down && unhandled))
        std::printf("  (down message received: %d, from the actor: %d, reason kind %d)\n",
                    (int)got, (int)down, reason_kind);
      auto r3 = self->request(mb, cafx::make_message(cafxg::mandel_tiles{{d}}), 30s);
      auto code_of = [](const auto& r) {
        return std::holds_alternative<cafx::error>(r) ? (int)std::get<cafx::error>(r).code : -1;
      };
      check(std::holds_alternative<cafx::message>(r1) &&
                std::get<cafx::message>(r1).get<cafxg::u32vec>(0) == expect_tile(d),
            "device loss: the request before the fault is answered exactly");
      check(code_of(r2) == (int)cafx::errc::request_down,
            "device loss: the faulting request gets error(request_down) (got " +
                std::to_string(code_of(r2)) + ")");
      check(down && unhandled, "device loss: monitors receive down(unhandled_error)");
      check(code_of(r3) == (int)cafx::errc::request_down,
            "device loss: later requests get request_down (got " + std::to_string(code_of(r3)) +
                ")");
      check(cafxg_ctx_status(lost_ctx) == CAFXG_E_DOWN, "device loss: ctx_status E_DOWN");
      cafxg_mandel_desc t = d;
      uint32_t out[4096];
      check(cafxg_mandelbrot(lost_ctx, &t, 1, out) == CAFXG_E_DOWN,
            "submissions on a lost context fail at once with request_down");
      // (the context is closed after the actor system: the actor object
      // may outlive this scope in a pending relay job)
    }
    // ~actor_system: hard-kills the gpu actors, which unregister (no hang)
  }
  std::printf("PASS actor_system shutdown with registered gpu actors\n");
  if (lost_ctx)
    cafxg_close(lost_ctx);
  cafxg_close(ctx);
  std::printf("%s\n", failures ? "FAILED" : "ALL PASS");
  return failures ? 1 : 0;
}
