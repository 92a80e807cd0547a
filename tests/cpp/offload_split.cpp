// The paper's CPU/GPU offload experiment (SURVEY.md §8f
// row 3) on the unmodified reference runtime + the B200 compute actor.
//
// One 1920x1080 Mandelbrot image over [-0.5,0.1] x [-0.7375,-0.1375] is
// divided between CPU row actors (cafx event-based actors on the reference's
// scheduler, one per row, each replying `(uint32 y, u32vec row)` like
// bench.cpp's row_worker) and one request to the GPU actor (cafxg::spawn_gpu)
// for the remaining rows. The GPU share goes 0 %, 10 %, ..., 100 %; for each
// share the run is repeated R times and the mean / standard deviation of
// three clocks are reported: total (send to last reply), CPU (until the last
// CPU row arrived) and GPU (until the GPU reply arrived) -- the three curves
// of the paper's figure. Both sides evaluate the same fp32 contract (pixel
// centres, the reference's operation order), so the assembled image is
// identical at every share: each run's FNV-1a checksum is checked against
// the all-GPU image and the tool exits non-zero on any mismatch.
//
// Usage: offload_split [--runs R] [--iters 120,1200] [--json]
// Built by tests/cpp/Makefile against the reference runtime compiled from its
// sources (oracle/_ref/libcafx_ref.so); run by tests/test_offload_split_gpu.py.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cafx/actor_system.hpp"
#include "cafx/detail/fnv.hpp"
#include "cafx/scoped_actor.hpp"
#include "cafxg/gpu_actor.hpp"

using namespace std::chrono_literals;
using clk = std::chrono::steady_clock;

namespace {

constexpr uint32_t kW = 1920, kH = 1080;
constexpr double kX0 = -0.5, kX1 = 0.1, kY0 = -0.7375, kY1 = -0.1375;

// c = lo + ((i + 0.5) * (hi - lo)) / n in fp64, then binary32 (cafxg.h)
float coord(double lo, double hi, uint32_t i, uint32_t n) {
  volatile double k = i + 0.5;
  volatile double q = k * (hi - lo);
  return (float)(lo + q / n);
}

// bench.cpp:367-379's cell in binary32 (built with -ffp-contract=off)
uint32_t cell(float cr, float ci, uint32_t max_iter) {
  float zr = 0.0f, zi = 0.0f;
  for (uint32_t i = 1; i <= max_iter; ++i) {
    float nr = zr * zr - zi * zi + cr;
    float ni = 2 * zr * zi + ci;
    zr = nr;
    zi = ni;
    if (zr * zr + zi * zi > 4.0f)
      return i;
  }
  return max_iter;
}

struct Stat {
  std::vector<double> v;
  double mean() const {
    double s = 0;
    for (double x : v) s += x;
    return v.empty() ? 0 : s / v.size();
  }
  double sd() const {
    if (v.size() < 2) return 0;
    double m = mean(), s = 0;
    for (double x : v) s += (x - m) * (x - m);
    return std::sqrt(s / (v.size() - 1));
  }
};

template <class Vec>
uint64_t fnv(const Vec& img) {
  uint64_t h = cafx::detail::fnv1a_seed;
  for (uint32_t c : img)
    h = cafx::detail::fnv1a_u32(h, c);
  return h;
}

cafxg_mandel_desc gpu_rows(uint32_t row0, uint32_t nrows, uint32_t max_iter) {
  cafxg_mandel_desc d{};
  d.x0 = kX0; d.x1 = kX1; d.y0 = kY0; d.y1 = kY1;
  d.width = kW; d.height = kH;
  d.row0 = row0; d.nrows = nrows;
  d.col0 = 0; d.ncols = kW;
  d.max_iter = max_iter;
  d.precision = CAFXG_FP32;
  d.sampling = CAFXG_CENTRE;
  return d;
}

}  // namespace

int main(int argc, char** argv) {
  int runs = 20;
  std::vector<uint32_t> iters{120, 1200};
  bool json = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--runs" && i + 1 < argc) {
      runs = std::max(1, atoi(argv[++i]));
    } else if (a == "--iters" && i + 1 < argc) {
      iters.clear();
      for (char* s = argv[++i]; *s;) {
        iters.push_back((uint32_t)strtoul(s, &s, 10));
        if (*s == ',') ++s;
      }
    } else if (a == "--json") {
      json = true;
    }
  }
  cafxg_ctx* ctx = nullptr;
  if (cafxg_open(1, &ctx) != CAFXG_OK) {
    std::fprintf(stderr, "cafxg_open: %s\n", cafxg_last_error());
    return 1;
  }
  int failures = 0;
  {
    cafx::actor_system sys;
    cafx::scoped_actor self{sys};
    auto gpu = cafxg::spawn_gpu(sys, ctx, "mandelbrot", {});
    const auto me = self.handle();
    std::vector<uint32_t> img((size_t)kW * kH);
    if (!json)
      std::printf("# %ux%u fp32 [%g,%g]x[%g,%g], %d runs per share, CPU = cafx row actors on "
                  "%u hardware threads, GPU = one B200 compute actor request\n",
                  kW, kH, kX0, kX1, kY0, kY1, runs, std::thread::hardware_concurrency());
    for (uint32_t it : iters) {
      // the all-GPU image is the reference for every share
      auto all = self->request(gpu, cafx::make_message(cafxg::mandel_tiles{{gpu_rows(0, kH, it)}}),
                               60s);
      if (!std::holds_alternative<cafx::message>(all)) {
        std::fprintf(stderr, "GPU request failed\n");
        failures++;
        break;
      }
      const uint64_t want = fnv(std::get<cafx::message>(all).get<cafxg::u32vec>(0));
      if (!json)
        std::printf("# max_iter %u (image checksum %016llx)\n%6s %12s %12s %12s %12s %12s %12s\n",
                    it, (unsigned long long)want, "gpu_%", "total_ms", "sd", "cpu_ms", "sd",
                    "gpu_ms", "sd");
      for (int share = 0; share <= 10; ++share) {
        const uint32_t g_rows = (uint32_t)std::lround(kH * share / 10.0);
        const uint32_t c_rows = kH - g_rows;
        Stat total, cpu, gpu_t;
        for (int r = -1; r < runs; ++r) {  // r = -1: warm-up
          std::fill(img.begin(), img.end(), 0u);
          auto t0 = clk::now();
          double t_cpu = 0, t_gpu = 0;
          if (g_rows)
            self->send(gpu, cafx::make_message(cafxg::mandel_tiles{{gpu_rows(c_rows, g_rows, it)}}));
          for (uint32_t y = 0; y < c_rows; ++y)
            sys.spawn([=](cafx::event_based_actor* worker) {
              cafxg::u32vec row(kW);
              const float ci = coord(kY0, kY1, y, kH);
              for (uint32_t x = 0; x < kW; ++x)
                row[x] = cell(coord(kX0, kX1, x, kW), ci, it);
              worker->send(me, cafx::make_message(y, std::move(row)));
            });
          uint32_t rows_left = c_rows;
          bool gpu_left = g_rows > 0;
          while (rows_left || gpu_left) {
            bool got = self->receive(
                cafx::behavior{
                    [&](uint32_t y, const cafxg::u32vec& row) {
                      std::memcpy(&img[(size_t)y * kW], row.data(), kW * 4);
                      if (--rows_left == 0)
                        t_cpu = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
                    },
                    [&](const cafxg::u32vec& counts) {
                      std::memcpy(&img[(size_t)c_rows * kW], counts.data(), counts.size() * 4);
                      gpu_left = false;
                      t_gpu = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
                    }},
                120s);
            if (!got) {
              std::fprintf(stderr, "timeout waiting for replies\n");
              return 1;
            }
          }
          double t_all = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
          if (fnv(img) != want) {
            std::fprintf(stderr, "checksum mismatch at max_iter %u share %d%%\n", it, share * 10);
            failures++;
          }
          if (r < 0)
            continue;
          total.v.push_back(t_all);
          if (c_rows) cpu.v.push_back(t_cpu);
          if (g_rows) gpu_t.v.push_back(t_gpu);
        }
        if (json)
          std::printf("{\"max_iter\": %u, \"gpu_share\": %d, \"runs\": %d, \"total_ms\": %.4f, "
                      "\"total_sd\": %.4f, \"cpu_ms\": %.4f, \"cpu_sd\": %.4f, \"gpu_ms\": %.4f, "
                      "\"gpu_sd\": %.4f, \"checksum_ok\": %s}\n",
                      it, share * 10, runs, total.mean(), total.sd(), cpu.mean(), cpu.sd(),
                      gpu_t.mean(), gpu_t.sd(), failures ? "false" : "true");
        else
          std::printf("%6d %12.3f %12.3f %12.3f %12.3f %12.3f %12.3f\n", share * 10, total.mean(),
                      total.sd(), cpu.mean(), cpu.sd(), gpu_t.mean(), gpu_t.sd());
        std::fflush(stdout);
      }
    }
  }
  cafxg_close(ctx);
  if (!json)
    std::printf("%s\n", failures ? "CHECKSUM MISMATCH" : "all shares produced the all-GPU image");
  return failures ? 1 : 0;
}
