// Device-side descriptors shared by the Mandelbrot kernels and the host
// runtime (rt_mandel.cpp, rt_actor.cpp).
#pragma once
#include <cstdint>

#include "dcheck.cuh"

namespace cafxg {

// One tile of a batch, as the kernel sees it. Built on the host from
// cafxg_mandel_desc (include/cafxg.h). Tiles are split into chunks of
// chunk_px pixels; chunks never straddle tiles, and chunk_begin is the global
// index of the tile's first chunk (ascending across the batch).
struct MTile {
  double x0, xspan, y0, yspan;  // xspan = x1 - x0, yspan = y1 - y0 (fp64)
  double s;                     // 0 (corner) or 0.5 (pixel centre)
  uint32_t width, height;       // full image, for the coordinate mapping
  uint32_t row0, col0;          // tile origin in the image
  uint32_t nrows, ncols;
  uint32_t max_iter;
  uint32_t chunk_begin;
  uint32_t chunks_per_row;      // ceil(ncols / chunk_px); chunks never straddle rows
  uint32_t out_off;             // tile's first count in MLaunch::out (row-major,
                                // pitch ncols); launch total < 2^32 elements
  // Coordinate tables (filled by the prologue kernel): cx[ncols] real parts
  // of the tile's columns, cy[nrows] imaginary parts of its rows, stored in
  // the request precision (float or double).
  void* cx;
  void* cy;
  // Direct reply (MLaunch::direct): the tile's reply buffer, device-mapped
  // pinned host memory, 16-byte aligned; the kernel copies the finished tile
  // there itself.
  uint32_t* reply;
};

constexpr int kInlineTiles = 32;   // tiles passed by value in the params (< 4 KB)
// Pixels per work chunk: one refill generation of a warp in fp32 (32 lanes x
// 4 slots), so when the cursor runs dry no warp still holds unstarted pixels
// (512-pixel chunks left ~0.2 ms tails per launch). fp64 warps have 2 slots
// per lane; 64-pixel chunks for them measured slower (fp64 reference mode
// 21.65 -> 21.9 ms, more cursor traffic) and no faster for small batches.
constexpr uint32_t kChunkPx = 128;
constexpr uint32_t chunk_px(int /*precision*/) { return kChunkPx; }
constexpr int kMandelThreads = 256;

struct MLaunch {
  MTile inl[kInlineTiles];
  const MTile* tiles;   // device copy when n > kInlineTiles
  uint32_t* out;        // counts of every tile (MTile::out_off)
  uint32_t n;
  uint32_t total_chunks;
  uint32_t max_iter;    // one max_iter per launch (the host splits batches)
  uint32_t* sched;      // [0] chunk cursor, [1] finished blocks (self-reset)
  float zero;           // always 0.0f; opaque to ptxas (see the escape block)
  uint32_t inline_coords;  // 1: tiles carry no coordinate tables (cx == cy == null)
  uint32_t block_reps;  // deferred kernel: unrolled units per unchecked block
  // Direct reply: n <= kInlineTiles tiles, each a multiple of 4 pixels at a
  // 4-pixel-aligned out_off, batch < 2^kDirectShift pixels. Output offsets then
  // carry the tile index in their top bits; tile_done[t] counts the tile's
  // finished pixels (zero at launch, reset by the warp that copies the tile).
  uint32_t direct;
  uint32_t* tile_done;
  uint64_t out_limit;   // elements of `out` the launch may write (checked build)
};
static_assert(sizeof(MLaunch) <= 4096, "MLaunch is passed by value");
constexpr int kDirectShift = 26;

// Host launchers (mandelbrot.cu). precision: 0 = fp32, 1 = fp64.
// `exact` selects the 8-op escape step; the default 7-op step folds
// 2*zr*zi + ci into fma(zr*zi, 2, ci), which is bit-identical whenever no
// row has 0 < |ci| < 2^-100 (fp32) / 2^-960 (fp64): see DESIGN.md §3.
// `deferred` selects mandel_deferred_kernel (escape tested once per block of
// ksteps, escaped blocks replayed; valid only when no tile reaches
// 2 - 2^-10 < |c| < 2 + 2^-10, see mandelbrot.cu).
struct MandelLaunchCfg {
  int grid;
  int ksteps;      // checked kernel: steps between refills (4 / 16 / 32)
  bool exact;
  bool deferred;
  int unit = 8;    // deferred kernel: unrolled steps per unit (8 or 32) ...
  int reps = 4;    // ... and units per unchecked block (block = unit x reps)
};
int mandel_launch(const MLaunch& L, int precision, const MandelLaunchCfg& cfg,
                  void* stream);
// Prologue: fills every tile's cx/cy tables (grid.y = tile).
int mandel_coords_launch(const MLaunch& L, int precision, uint32_t max_extent,
                         void* stream);
int mandel_max_blocks_per_sm(int precision, int ksteps, bool exact, bool deferred, int unit);
int mandel_slots_per_thread(int precision);

}  // namespace cafxg
