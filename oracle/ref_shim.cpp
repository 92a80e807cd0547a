// TEST INFRASTRUCTURE ONLY -- C entry points into the UNMODIFIED reference
// (compiled from /root/reference/proj sources by oracle/Makefile into
// oracle/_ref/libcafx_ref.so). Used by tests/golden/make_golden.py to pin the
// oracle, and by bench.py's reference arm for the paper-scale CPU number.
//
//   ref_mandelbrot_cell -> cafx::bench::mandelbrot_cell  bench.cpp:367
//   ref_mandelbrot_row  -> cafx::bench::mandelbrot_row   bench.cpp:381
//   ref_run_mandelbrot  -> cafx::bench::run_mandelbrot   bench.cpp:481
//   ref_region_iters_mt -> cafx::bench::mandelbrot_cell over a sampled region
//                          (the CPU baseline of bench.py on BASELINE cfg3)
//   ref_tiles_mt        -> cafx::bench::mandelbrot_cell over every pixel of a
//                          list of tiles (bench.py's cfg4 CPU baseline and
//                          the per-tile check of every storm reply)
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "cafx/bench/bench.hpp"

extern "C" {

uint32_t ref_mandelbrot_cell(double re, double im, uint32_t max_iter) {
  return cafx::bench::mandelbrot_cell(re, im, max_iter);
}

void ref_mandelbrot_row(uint32_t y, uint32_t size, uint32_t max_iter,
                        uint32_t* out) {
  auto row = cafx::bench::mandelbrot_row(y, size, max_iter);
  std::memcpy(out, row.data(), row.size() * sizeof(uint32_t));
}

uint64_t ref_run_mandelbrot(uint32_t size, uint32_t max_iter,
                            uint32_t workers, double* wall_clock_ms) {
  cafx::bench::bench_options opts;
  opts.workers = workers;
  auto report = cafx::bench::run_mandelbrot(size, max_iter, opts);
  if (wall_clock_ms)
    *wall_clock_ms = report.wall_clock_ms;
  return report.checksum;
}

// The reference's own escape-time function (fp64: the reference has no fp32)
// over every row_stride-th row of a W x H region sampled at pixel centres
// (c = lo + ((i + 0.5) * span) / n, the generalised mapping of SURVEY.md
// §8a row a2), rows dealt cyclically to `threads` threads. Returns the sum of
// the counts; *seconds = wall time of the parallel region.
uint64_t ref_region_iters_mt(double x0, double x1, double y0, double y1, uint32_t width,
                             uint32_t height, uint32_t max_iter, uint32_t row_stride,
                             uint32_t threads, double* seconds) {
  if (row_stride == 0)
    row_stride = 1;
  if (threads == 0)
    threads = 1;
  std::vector<uint64_t> part(threads, 0);
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < threads; ++t) {
    th.emplace_back([&, t] {
      uint64_t sum = 0;
      uint32_t k = 0;
      for (uint32_t y = 0; y < height; y += row_stride, ++k) {
        if (k % threads != t)
          continue;
        const double im = y0 + (((double)y + 0.5) * (y1 - y0)) / height;
        for (uint32_t x = 0; x < width; ++x) {
          const double re = x0 + (((double)x + 0.5) * (x1 - x0)) / width;
          sum += cafx::bench::mandelbrot_cell(re, im, max_iter);
        }
      }
      part[t] = sum;
    });
  }
  for (auto& x : th)
    x.join();
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  uint64_t total = 0;
  for (uint64_t v : part)
    total += v;
  return total;
}

// Tile records with the memory layout of cafxg_mandel_desc (include/cafxg.h):
// the generalised mapping c = lo + ((i + s) * (hi - lo)) / n in fp64 (s = 0.5
// at pixel centres), counts by the reference's own mandelbrot_cell (fp64, the
// reference's only precision). Tiles are packed in order into `out` (nrows x
// ncols each, row-major) and claimed by `threads` threads one at a time.
// Returns the sum of the counts; *seconds = wall time of the parallel region.
struct ref_tile {
  double x0, x1, y0, y1;
  uint32_t width, height, row0, nrows, col0, ncols, max_iter, precision, sampling, reserved;
  uint64_t out_offset;
};
static_assert(sizeof(ref_tile) == 80, "layout of cafxg_mandel_desc");

uint64_t ref_tiles_mt(const ref_tile* tiles, size_t n, uint32_t* out, uint32_t threads,
                      double* seconds) {
  if (threads == 0)
    threads = 1;
  std::vector<uint64_t> off(n + 1, 0);
  for (size_t i = 0; i < n; ++i)
    off[i + 1] = off[i] + (uint64_t)tiles[i].nrows * tiles[i].ncols;
  std::atomic<size_t> next{0};
  std::vector<uint64_t> part(threads, 0);
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < threads; ++t) {
    th.emplace_back([&, t] {
      uint64_t sum = 0;
      for (size_t i = next++; i < n; i = next++) {
        const ref_tile& d = tiles[i];
        const double s = d.sampling ? 0.5 : 0.0;
        uint32_t* o = out + off[i];
        for (uint32_t r = 0; r < d.nrows; ++r) {
          const double im = d.y0 + (((double)(d.row0 + r) + s) * (d.y1 - d.y0)) / d.height;
          for (uint32_t c = 0; c < d.ncols; ++c) {
            const double re = d.x0 + (((double)(d.col0 + c) + s) * (d.x1 - d.x0)) / d.width;
            const uint32_t k = cafx::bench::mandelbrot_cell(re, im, d.max_iter);
            o[(size_t)r * d.ncols + c] = k;
            sum += k;
          }
        }
      }
      part[t] = sum;
    });
  }
  for (auto& x : th)
    x.join();
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  uint64_t total = 0;
  for (uint64_t v : part)
    total += v;
  return total;
}

} // extern "C"
