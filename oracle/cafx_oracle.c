/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the cafx-b200 compute-actor path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library, and only as the checker or
 * as the reported CPU baseline. The product path (libcafxg.so) never links,
 * loads or falls back to it.
 *
 * This is a restatement (not a copy) of the reference's Mandelbrot hot path:
 *   - mandelbrot_cell   /root/reference/proj/src/bench/bench.cpp:367-379
 *   - mandelbrot_row    /root/reference/proj/src/bench/bench.cpp:381-390
 *   - collector FNV     /root/reference/proj/src/bench/bench.cpp:326-333
 *   - fnv1a / fnv1a_u32 /root/reference/proj/include/cafx/detail/fnv.hpp:8-28
 *   - run_mandelbrot    /root/reference/proj/src/bench/bench.cpp:481-505
 *     (one task per row, rows hashed in y order by one collector)
 * generalised to rectangular images, arbitrary regions,
 * pixel-centre sampling and fp32. Reference mode (x0=-1.5, x1=0.5, y0=-1,
 * y1=1, corner sampling, W=H=size, fp64) is bit-identical to bench.cpp.
 *
 * Parity pin: tests/test_oracle.py checks this file against the golden
 * checksums produced by the reference itself (oracle/_ref, built from the
 * reference sources by oracle/Makefile) and the pins of the reference's own
 * tests (test_bench.cpp:76-82, acceptance.cpp:632-672).
 *
 * Must be compiled with -ffp-contract=off: the reference binary has no FMA
 * contraction (built -O3 without -march, SURVEY.md §2 "Build").
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_FNV_SEED 0xcbf29ce484222325ull
#define ORACLE_FNV_PRIME 0x100000001b3ull

/* ---- escape-time cells (bench.cpp:367-379) ------------------------------- */

uint32_t oracle_cell_f64(double re, double im, uint32_t max_iter) {
  double zr = 0.0, zi = 0.0;
  for (uint32_t i = 1; i <= max_iter; ++i) {
    double nr = zr * zr - zi * zi + re;
    double ni = 2 * zr * zi + im;
    zr = nr;
    zi = ni;
    if (zr * zr + zi * zi > 4.0)
      return i;
  }
  return max_iter;
}

/* Same operation order, evaluated in binary32 (FLT_EVAL_METHOD == 0). */
uint32_t oracle_cell_f32(float re, float im, uint32_t max_iter) {
  float zr = 0.0f, zi = 0.0f;
  for (uint32_t i = 1; i <= max_iter; ++i) {
    float nr = zr * zr - zi * zi + re;
    float ni = 2 * zr * zi + im;
    zr = nr;
    zi = ni;
    if (zr * zr + zi * zi > 4.0f)
      return i;
  }
  return max_iter;
}

/* ---- coordinate mapping (generalised contract) ------
 * c = lo + ((i + s) * (hi - lo)) / n, evaluated in fp64, multiply before
 * divide; s = 0 (corner, reference mode) or 0.5 (pixel centre). In reference
 * mode (lo=-1.5, hi-lo=2.0, s=0) this equals bench.cpp:386's
 * `2.0 * x / size - 1.5` bit for bit. */
double oracle_coord(double lo, double hi, uint32_t i, uint32_t n, int centre) {
  double k = (double)i + (centre ? 0.5 : 0.0);
  return lo + (k * (hi - lo)) / (double)n;
}

/* ---- rows (bench.cpp:381-390) -------------------------------------------- */

void oracle_mandelbrot_row(uint32_t y, uint32_t size, uint32_t max_iter,
                           uint32_t* out) {
  double ci = 2.0 * y / size - 1.0;
  for (uint32_t x = 0; x < size; ++x) {
    double cr = 2.0 * x / size - 1.5;
    out[x] = oracle_cell_f64(cr, ci, max_iter);
  }
}

/* Tile of a generalised request: rows [row0,row0+nrows) x cols
 * [col0,col0+ncols) of a width x height image over [x0,x1] x [y0,y1]; output
 * row-major with pitch ncols. precision: 0 = fp32, 1 = fp64. */
typedef struct {
  double x0, x1, y0, y1;
  uint32_t width, height;
  uint32_t row0, nrows, col0, ncols;
  uint32_t max_iter;
  uint32_t precision;
  uint32_t centre;
} oracle_tile;

static void tile_rows(const oracle_tile* t, uint32_t r_begin, uint32_t r_end,
                      uint32_t r_step, uint32_t* out) {
  for (uint32_t r = r_begin; r < r_end; r += r_step) {
    uint32_t* dst = out + (size_t)r * t->ncols;
    double ci = oracle_coord(t->y0, t->y1, t->row0 + r, t->height, t->centre);
    for (uint32_t c = 0; c < t->ncols; ++c) {
      double cr = oracle_coord(t->x0, t->x1, t->col0 + c, t->width, t->centre);
      dst[c] = t->precision
                 ? oracle_cell_f64(cr, ci, t->max_iter)
                 : oracle_cell_f32((float)cr, (float)ci, t->max_iter);
    }
  }
}

void oracle_mandelbrot_tile(const oracle_tile* t, uint32_t* out) {
  tile_rows(t, 0, t->nrows, 1, out);
}

/* ---- FNV-1a over big-endian cells (fnv.hpp:23-28, bench.cpp:329-331) ----- */

uint64_t oracle_fnv1a_u32(uint64_t h, const uint32_t* cells, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t x = cells[i];
    h = (h ^ (uint8_t)(x >> 24)) * ORACLE_FNV_PRIME;
    h = (h ^ (uint8_t)(x >> 16)) * ORACLE_FNV_PRIME;
    h = (h ^ (uint8_t)(x >> 8)) * ORACLE_FNV_PRIME;
    h = (h ^ (uint8_t)x) * ORACLE_FNV_PRIME;
  }
  return h;
}

uint64_t oracle_fnv_seed(void) {
  return ORACLE_FNV_SEED;
}

/* ---- threaded drivers ------------------------------------------------------
 * The reference spawns one actor per row on a work-stealing scheduler
 * (bench.cpp:494-495); the oracle deals rows cyclically to `threads` pthreads,
 * which is the same decomposition without the runtime. */

typedef struct {
  const oracle_tile* tile;
  uint32_t* out;
  uint32_t first, step, stride;
} tile_job;

static void* tile_worker(void* arg) {
  tile_job* j = (tile_job*)arg;
  tile_rows(j->tile, j->first, j->tile->nrows, j->step, j->out);
  return NULL;
}

/* Computes every `sample_stride`-th row (1 = all rows) with `threads`
 * threads; returns the number of rows computed. */
uint32_t oracle_mandelbrot_tile_mt(const oracle_tile* t, uint32_t* out,
                                   uint32_t threads, uint32_t sample_stride) {
  if (threads == 0)
    threads = 1;
  if (sample_stride == 0)
    sample_stride = 1;
  pthread_t* tids = (pthread_t*)calloc(threads, sizeof(pthread_t));
  tile_job* jobs = (tile_job*)calloc(threads, sizeof(tile_job));
  for (uint32_t k = 0; k < threads; ++k) {
    jobs[k].tile = t;
    jobs[k].out = out;
    jobs[k].first = k * sample_stride;
    jobs[k].step = threads * sample_stride;
    pthread_create(&tids[k], NULL, tile_worker, &jobs[k]);
  }
  for (uint32_t k = 0; k < threads; ++k)
    pthread_join(tids[k], NULL);
  free(tids);
  free(jobs);
  uint32_t rows = 0;
  for (uint32_t r = 0; r < t->nrows; r += sample_stride)
    ++rows;
  return rows;
}

/* run_mandelbrot(size, max_iter) checksum (bench.cpp:481-505 + the collector
 * at :326-333): all rows, reference area, fp64, rows hashed in y order. */
uint64_t oracle_run_mandelbrot(uint32_t size, uint32_t max_iter,
                               uint32_t threads) {
  oracle_tile t = {-1.5, 0.5, -1.0, 1.0, size, size, 0, size, 0, size,
                   max_iter, 1, 0};
  uint32_t* out = (uint32_t*)malloc((size_t)size * size * sizeof(uint32_t));
  oracle_mandelbrot_tile_mt(&t, out, threads, 1);
  uint64_t h = oracle_fnv1a_u32(ORACLE_FNV_SEED, out, (size_t)size * size);
  free(out);
  return h;
}

uint64_t oracle_sum_u32(const uint32_t* cells, size_t n) {
  uint64_t s = 0;
  for (size_t i = 0; i < n; ++i)
    s += cells[i];
  return s;
}
