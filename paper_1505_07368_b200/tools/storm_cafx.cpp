// BASELINE config 4 through the drop-in itself: 64 cafx event-based client
// actors on the UNMODIFIED reference runtime (oracle/_ref/libcafx_ref.so)
// send their 1600 storm tiles each to one gpu_actor (include/cafxg/
// gpu_actor.hpp) and check every reply. Timed by bench.py.
//
//   storm_cafx <descs.bin> <expect.u32> <clients> <per> <closed|open> [device_mask]
//              [steal_sleep_us]
//
// descs.bin: clients*per cafxg_mandel_desc records (client c owns records
// [c*per, (c+1)*per)); expect.u32: the same number of 64x64 tiles of
// expected counts (computed by the reference's own mandelbrot_cell on the
// CPU, bench.py), row-major, packed in record order.
//
//  closed: each client chains sync_send(...).then(...) (one outstanding
//          request, local_actor.cpp:66-115); a reply is compared with its
//          tile's expected counts byte for byte (memcmp) in the handler.
//  open:   each client sends all its requests at once with async `send`
//          (local_actor.cpp:56-64, the reply goes to the sender's mailbox,
//          local_actor.cpp:319-329); async replies carry no request id, so
//          each reply's 64-bit fingerprint (weighted word sum) is recorded
//          and, after the run, the multiset of a client's reply fingerprints
//          must equal that of its expected tiles.
//
// One untimed warm-up storm of the same shape runs first (pinned reply pool,
// staging ring, first launches). Prints one JSON line.
//
// steal_sleep_us sets the reference scheduler's idle back-off
// (scheduler_config::steal_sleep, scheduler.hpp:33; default 1000 us): an idle
// cafx worker polls its deque and sleeps that long between sweeps
// (scheduler.hpp:374-402), and a reply delivered from a backend thread waits
// in a worker's deque until the worker wakes, so closed-loop round trips are
// bounded below by it. Omitted = the reference's default configuration.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "cafx/actor_system.hpp"
#include "cafx/scheduler.hpp"
#include "cafx/scoped_actor.hpp"
#include "cafxg/gpu_actor.hpp"

using namespace std::chrono_literals;

namespace {

constexpr size_t kTilePx = 64 * 64;

const void* map_file(const char* path, size_t bytes) {
  int fd = open(path, O_RDONLY);
  if (fd < 0)
    return nullptr;
  struct stat st {};
  if (fstat(fd, &st) != 0 || (size_t)st.st_size < bytes) {
    close(fd);
    return nullptr;
  }
  void* p = mmap(nullptr, bytes, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
  close(fd);
  return p == MAP_FAILED ? nullptr : p;
}

// 64-bit fingerprint of one tile: sum of its 64-bit words times fixed odd
// weights (vectorises; a wrong reply collides with probability ~2^-64)
uint64_t fingerprint(const uint32_t* t) {
  const uint64_t* w = reinterpret_cast<const uint64_t*>(t);
  uint64_t h = 0;
  for (size_t i = 0; i < kTilePx / 2; ++i)
    h += w[i] * (0x9e3779b97f4a7c15ull + 2 * i);
  return h;
}

struct Run {
  const cafxg_mandel_desc* descs;
  const uint32_t* expect;
  int clients, per;
  bool open_loop;
  std::atomic<int> finished{0};
  std::atomic<uint64_t> good{0}, bad{0}, errors{0};
  std::vector<std::vector<uint64_t>> prints;  // open loop, per client
};

double storm(cafx::actor_system& sys, const cafx::actor& mb, Run& run) {
  run.finished = 0;
  run.good = run.bad = run.errors = 0;
  run.prints.assign(run.clients, {});
  std::vector<cafx::actor> clients;
  clients.reserve(run.clients);
  for (int c = 0; c < run.clients; ++c) {
    Run* R = &run;
    if (!run.open_loop) {
      clients.push_back(sys.spawn([R, c, mb](cafx::event_based_actor* me) {
        return cafx::behavior{
            [R, c, mb, me](uint32_t k) {
              const size_t idx = (size_t)c * R->per + k;
              cafx::actor self_handle{cafx::abstract_actor_ptr{me}};
              me->sync_send(mb, cafx::make_message(cafxg::mandel_tiles{{R->descs[idx]}}))
                  .then(
                      [R, c, k, idx, me, self_handle](const cafxg::u32vec& counts) {
                        const bool ok = counts.size() == kTilePx &&
                                        std::memcmp(counts.data(), R->expect + idx * kTilePx,
                                                    kTilePx * 4) == 0;
                        (ok ? R->good : R->bad)++;
                        if (k + 1 < (uint32_t)R->per) {
                          me->send(self_handle, cafx::make_message(k + 1));
                        } else {
                          R->finished++;
                          me->quit();
                        }
                      },
                      [R, me](const cafx::error&) {
                        R->errors++;
                        R->finished++;
                        me->quit();
                      });
            },
        };
      }));
    } else {
      run.prints[c].reserve(run.per);
      clients.push_back(sys.spawn([R, c, mb](cafx::event_based_actor* me) {
        return cafx::behavior{
            [R, c, mb, me](uint32_t) {
              for (int k = 0; k < R->per; ++k)
                me->send(mb, cafx::make_message(
                                 cafxg::mandel_tiles{{R->descs[(size_t)c * R->per + k]}}));
            },
            [R, c, me](const cafxg::u32vec& counts) {
              auto& v = R->prints[c];
              v.push_back(counts.size() == kTilePx ? fingerprint(counts.data()) : 0);
              if ((int)v.size() == R->per) {
                R->finished++;
                me->quit();
              }
            },
            [R, me](const cafx::error&) {
              R->errors++;
              R->finished++;
              me->quit();
            },
        };
      }));
    }
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (auto& cl : clients)
    sys.anon_send(cl, cafx::make_message(uint32_t{0}));
  while (run.finished.load(std::memory_order_acquire) < run.clients) {
    if (std::chrono::steady_clock::now() - t0 > 300s)
      break;
    std::this_thread::sleep_for(20us);
  }
  const double ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (run.open_loop) {
    // every client's replies == its expected tiles, as multisets
    for (int c = 0; c < run.clients; ++c) {
      std::vector<uint64_t> want(run.per);
      for (int k = 0; k < run.per; ++k)
        want[k] = fingerprint(run.expect + ((size_t)c * run.per + k) * kTilePx);
      auto got = run.prints[c];
      std::sort(want.begin(), want.end());
      std::sort(got.begin(), got.end());
      size_t i = 0, j = 0, match = 0;
      while (i < want.size() && j < got.size()) {
        if (want[i] == got[j]) {
          ++match, ++i, ++j;
        } else if (want[i] < got[j]) {
          ++i;
        } else {
          ++j;
        }
      }
      run.good += match;
      run.bad += got.size() - match;
    }
  }
  return ms;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s descs.bin expect.u32 clients per closed|open [mask]\n",
                 argv[0]);
    return 2;
  }
  Run run;
  run.clients = std::atoi(argv[3]);
  run.per = std::atoi(argv[4]);
  run.open_loop = std::string(argv[5]) == "open";
  const uint64_t mask = argc > 6 ? std::strtoull(argv[6], nullptr, 0) : 1;
  cafx::scheduler_config cfg = cafx::scheduler_config::from_env();
  if (argc > 7)
    cfg.steal_sleep = std::chrono::microseconds(std::atoll(argv[7]));
  const size_t total = (size_t)run.clients * run.per;
  run.descs = static_cast<const cafxg_mandel_desc*>(
      map_file(argv[1], total * sizeof(cafxg_mandel_desc)));
  run.expect = static_cast<const uint32_t*>(map_file(argv[2], total * kTilePx * 4));
  if (!run.descs || !run.expect) {
    std::fprintf(stderr, "storm_cafx: cannot map the descriptor / expectation files\n");
    return 2;
  }
  cafxg_ctx* ctx = nullptr;
  if (cafxg_open(mask, &ctx) != CAFXG_OK) {
    std::fprintf(stderr, "storm_cafx: cafxg_open: %s\n", cafxg_last_error());
    return 1;
  }
  double ms = 0;
  cafxg_stats s0{}, s1{};
  unsigned workers = 0;
  {
    workers = (unsigned)cfg.effective_workers();
    cafx::actor_system sys{cfg};
    auto mb = cafxg::spawn_gpu(sys, ctx, "mandelbrot", {});
    storm(sys, mb, run);  // warm-up
    cafxg_get_stats(ctx, &s0);
    ms = storm(sys, mb, run);
    cafxg_get_stats(ctx, &s1);
  }  // ~actor_system hard-kills the compute actor, which unregisters
  std::printf(
      "{\"mode\": \"%s\", \"clients\": %d, \"requests\": %zu, \"wall_ms\": %.3f, "
      "\"requests_per_s\": %.1f, \"good\": %llu, \"bad\": %llu, \"errors\": %llu, "
      "\"batches\": %llu, \"kernel_launches\": %llu, \"scheduler_workers\": %u, "
      "\"steal_sleep_us\": %lld, \"devices\": %d}\n",
      run.open_loop ? "open" : "closed", run.clients, total, ms, total / (ms / 1e3),
      (unsigned long long)run.good.load(), (unsigned long long)run.bad.load(),
      (unsigned long long)run.errors.load(), (unsigned long long)(s1.batches - s0.batches),
      (unsigned long long)(s1.kernel_launches - s0.kernel_launches), workers,
      (long long)cfg.steal_sleep.count(), cafxg_device_count(ctx));
  cafxg_close(ctx);
  return run.good.load() == total && run.errors.load() == 0 ? 0 : 3;
}
