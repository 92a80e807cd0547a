// TEST INFRASTRUCTURE ONLY -- C entry points into the UNMODIFIED reference
// (compiled from /root/reference/proj sources by oracle/Makefile into
// oracle/_ref/libcafx_ref.so). Used by tests/golden/make_golden.py to pin the
// oracle, and by bench.py's reference arm for the paper-scale CPU number.
//
//   ref_mandelbrot_cell -> cafx::bench::mandelbrot_cell  bench.cpp:367
//   ref_mandelbrot_row  -> cafx::bench::mandelbrot_row   bench.cpp:381
//   ref_run_mandelbrot  -> cafx::bench::run_mandelbrot   bench.cpp:481
#include <cstdint>
#include <cstring>

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

} // extern "C"
