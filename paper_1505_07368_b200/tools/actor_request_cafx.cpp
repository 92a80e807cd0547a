// cfg1 and cfg3 as single compute-actor requests through the drop-in itself:
// a cafx scoped_actor on the UNMODIFIED reference runtime requests one
// mandel_tiles message from a gpu_actor (include/cafxg/gpu_actor.hpp) and
// blocks on the reply (scoped_actor::request, scoped_actor.hpp:23-34).
// The reply vector is pinned pool memory the device writes into directly.
// Timed by bench.py next to the C-ABI end-to-end numbers.
//
//   actor_request_cafx [device_mask]
//
// Prints one JSON line: per config the median request-to-reply wall time,
// and the FNV-1a of the reply (fnv.hpp:23-28) so bench.py can compare the
// reply bit for bit with the C-ABI result / the oracle.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <variant>
#include <vector>

#include "cafx/actor_system.hpp"
#include "cafx/detail/fnv.hpp"
#include "cafx/scoped_actor.hpp"
#include "cafxg/gpu_actor.hpp"

using namespace std::chrono_literals;

namespace {

cafxg_mandel_desc desc(double x0, double x1, double y0, double y1, uint32_t w, uint32_t h,
                       uint32_t it) {
  cafxg_mandel_desc d{};
  d.x0 = x0; d.x1 = x1; d.y0 = y0; d.y1 = y1;
  d.width = d.ncols = w;
  d.height = d.nrows = h;
  d.max_iter = it;
  d.precision = CAFXG_FP32;
  d.sampling = CAFXG_CENTRE;
  return d;
}

struct Result {
  double median_ms = -1, min_ms = -1;
  uint64_t fnv = 0;
  bool ok = false;
};

Result time_requests(cafx::scoped_actor& self, const cafx::actor& mb, const cafxg_mandel_desc& d,
                     int reps) {
  Result r;
  std::vector<double> ms;
  for (int i = 0; i <= reps; ++i) {  // the first request is the warm-up
    cafxg::mandel_tiles req{{d}};
    auto msg = cafx::make_message(std::move(req));
    const auto t0 = std::chrono::steady_clock::now();
    auto res = self->request(mb, std::move(msg), 300s);
    const double dt =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (!std::holds_alternative<cafx::message>(res))
      return r;
    if (i > 0)
      ms.push_back(dt);
    if (i == reps) {
      const auto& counts = std::get<cafx::message>(res).get<cafxg::u32vec>(0);
      uint64_t h = cafx::detail::fnv1a_seed;
      for (uint32_t c : counts)
        h = cafx::detail::fnv1a_u32(h, c);
      r.fnv = h;
      r.ok = counts.size() == (size_t)d.nrows * d.ncols;
    }
  }
  std::sort(ms.begin(), ms.end());
  r.median_ms = ms[ms.size() / 2];
  r.min_ms = ms.front();
  return r;
}

}  // namespace

int main(int argc, char** argv) {
  const uint64_t mask = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : 1;
  cafxg_ctx* ctx = nullptr;
  if (cafxg_open(mask, &ctx) != CAFXG_OK) {
    std::fprintf(stderr, "actor_request_cafx: cafxg_open: %s\n", cafxg_last_error());
    return 1;
  }
  Result r1, r3;
  {
    cafx::actor_system sys;
    cafx::scoped_actor self{sys};
    auto mb = cafxg::spawn_gpu(sys, ctx, "mandelbrot", {});
    r1 = time_requests(self, mb, desc(-2.0, 1.0, -1.0, 1.0, 1920, 1080, 100), 30);
    r3 = time_requests(self, mb, desc(-0.75, -0.73, 0.10, 0.12, 16384, 16384, 1000), 3);
  }
  std::printf(
      "{\"cfg1\": {\"median_ms\": %.4f, \"min_ms\": %.4f, \"fnv\": \"%llu\", \"ok\": %s}, "
      "\"cfg3\": {\"median_ms\": %.3f, \"min_ms\": %.3f, \"fnv\": \"%llu\", \"ok\": %s}, "
      "\"devices\": %d}\n",
      r1.median_ms, r1.min_ms, (unsigned long long)r1.fnv, r1.ok ? "true" : "false",
      r3.median_ms, r3.min_ms, (unsigned long long)r3.fnv, r3.ok ? "true" : "false",
      cafxg_device_count(ctx));
  cafxg_close(ctx);
  return r1.ok && r3.ok ? 0 : 3;
}
