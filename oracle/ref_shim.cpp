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

} // extern "C"
