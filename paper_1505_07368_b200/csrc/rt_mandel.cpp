// libcafxg.so host runtime, Mandelbrot: request validation, the step
// choice, launch configuration, the multi-device row-band planner, host
// requests in overlapped waves, and the Mandelbrot / FNV / run_mandelbrot
// entry points of the C ABI.
#include "runtime_internal.hpp"

namespace cafxg {

// ---- Mandelbrot planning -----------------------------------------------------------

int validate_mandel(const cafxg_mandel_desc& t) {
  if (!std::isfinite(t.x0) || !std::isfinite(t.x1) || !std::isfinite(t.y0) ||
      !std::isfinite(t.y1))
    return fail(CAFXG_E_CONFIG, "mandelbrot: region must be finite");
  if (t.width == 0 || t.height == 0)
    return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot: empty image");
  if ((uint64_t)t.row0 + t.nrows > t.height || (uint64_t)t.col0 + t.ncols > t.width)
    return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot: tile outside the image");
  if (t.precision > 1 || t.sampling > 1)
    return fail(CAFXG_E_CONFIG, "mandelbrot: bad precision or sampling");
  if (t.max_iter > (1u << 30))
    return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot: max_iter above 2^30");
  if ((uint64_t)t.nrows * t.ncols > 0xffffffffull)
    return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot: tile above 2^32 pixels");
  return CAFXG_OK;
}

double coord(double lo, double hi, uint32_t i, uint32_t n, double s) {
  volatile double k = (double)i + s;  // volatile: keep every rounding explicit
  volatile double p = k * (hi - lo);
  volatile double q = p / (double)n;
  return lo + q;
}

// Smallest nonzero |ci| the tile's rows produce, in the request precision.
// The map row -> ci is monotone, so the minimum sits next to the zero
// crossing or at an end row.
double min_abs_ci(const cafxg_mandel_desc& t) {
  double s = t.sampling ? 0.5 : 0.0;
  int64_t cand[8] = {(int64_t)t.row0, (int64_t)t.row0 + t.nrows - 1};
  int nc = 2;
  double span = t.y1 - t.y0;
  if (span != 0.0) {
    double r = -t.y0 * (double)t.height / span - s;
    if (std::isfinite(r) && std::fabs(r) < 9.0e18) {
      for (int64_t k = (int64_t)std::floor(r) - 2; k <= (int64_t)std::floor(r) + 3; ++k)
        cand[nc++] = k;
    }
  }
  double best = INFINITY;
  for (int i = 0; i < nc; ++i) {
    const int64_t r = cand[i];
    if (r < (int64_t)t.row0 || r >= (int64_t)t.row0 + t.nrows)
      continue;
    double ci = coord(t.y0, t.y1, (uint32_t)r, t.height, s);
    double v = t.precision ? std::fabs(ci) : std::fabs((double)(float)ci);
    if (v > 0.0 && v < best)
      best = v;
  }
  return best;
}

// The 7-op escape step is bit-identical unless a row has a tiny nonzero ci
// (DESIGN.md §3): fp32 needs |ci| >= 2^-100, fp64 |ci| >= 2^-960.
bool needs_exact_step(const cafxg_mandel_desc& t);
bool use_exact(cafxg_ctx* ctx, const cafxg_mandel_desc& t) {
  return ctx->force_exact || needs_exact_step(t);
}
bool needs_exact_step(const cafxg_mandel_desc& t) {
  double lim = t.precision ? std::ldexp(1.0, -960) : std::ldexp(1.0, -100);
  return min_abs_ci(t) < lim;
}

// Work chunks of a tile: rows x ceil(ncols / chunk) (chunks never straddle
// rows, see mandel_kernel); a chunk is one refill generation of a warp.
uint32_t tile_chunks(uint32_t nrows, uint32_t ncols, uint32_t precision) {
  const uint32_t c = chunk_px((int)precision);
  return nrows * ((ncols + c - 1) / c);
}

void fill_mtile(MTile& m, const cafxg_mandel_desc& d, uint64_t out_off,
                       uint32_t chunk_begin) {
  m.x0 = d.x0;
  m.xspan = d.x1 - d.x0;
  m.y0 = d.y0;
  m.yspan = d.y1 - d.y0;
  m.s = d.sampling ? 0.5 : 0.0;
  m.width = d.width;
  m.height = d.height;
  m.row0 = d.row0;
  m.col0 = d.col0;
  m.nrows = d.nrows;
  m.ncols = d.ncols;
  m.max_iter = d.max_iter;
  m.chunk_begin = chunk_begin;
  m.chunks_per_row = (d.ncols + chunk_px((int)d.precision) - 1) / chunk_px((int)d.precision);
  m.out_off = (uint32_t)out_off;
  m.cx = m.cy = nullptr;
  m.reply = nullptr;
}

// Precondition of the deferred escape test (mandel_deferred_kernel): the
// tile's coordinate box stays outside the annulus 2 - 2^-10 < |c| < 2 + 2^-10,
// where an orbit could pass the reference's test and fall back below it.
bool deferred_safe(const MTile& t) {
  auto at = [](double lo, double span, double s, uint32_t i, uint32_t n) {
    return lo + (((double)i + s) * span) / n;
  };
  double xa = at(t.x0, t.xspan, t.s, t.col0, t.width);
  double xb = at(t.x0, t.xspan, t.s, t.col0 + t.ncols - 1, t.width);
  double ya = at(t.y0, t.yspan, t.s, t.row0, t.height);
  double yb = at(t.y0, t.yspan, t.s, t.row0 + t.nrows - 1, t.height);
  if (xa > xb) std::swap(xa, xb);
  if (ya > yb) std::swap(ya, yb);
  const double dx = xa > 0 ? xa : (xb < 0 ? -xb : 0.0);
  const double dy = ya > 0 ? ya : (yb < 0 ? -yb : 0.0);
  const double rmin = std::hypot(dx, dy);
  const double rmax = std::hypot(std::max(std::fabs(xa), std::fabs(xb)),
                                 std::max(std::fabs(ya), std::fabs(yb)));
  const double eta = std::ldexp(1.0, -10), pad = 1e-6;  // pad: fp32 rounding of c
  return rmax < 2.0 - eta - pad || rmin > 2.0 + eta + pad;
}

// CAFXG_DIRECT_REPLY=0 keeps every batch on the reply-scatter launch
bool direct_reply_enabled() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_DIRECT_REPLY");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CAFXG_DEFERRED=0 forces the per-step-checked kernel everywhere
bool deferred_enabled() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_DEFERRED");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Unchecked block length B of the deferred kernel. Modelled cost per pixel
// that never escapes, relative to max_iter steps:
//   ceil(max_iter / B) * B / max_iter * (1 + alpha / B) + gamma * B
// (overshoot past max_iter; block-end test and refill, ~alpha steps' worth;
// replays of escaped blocks grow with B). alpha = 7 (fp32) / 2 (fp64: the
// steps cost twice as much) and gamma = 0.002 fit the block-length sweep
// (DESIGN.md §3.1): cfg3 (fp32, max_iter 1000) runs 38.0 / 35.7 / 35.2 /
// 34.9 / 35.0 ms at B = 32 / 40 / 48 / 56 / 64 and picks 56; the fp64
// reference mode (max_iter 500) picks 24. Each B is one fully unrolled PTX
// block (8-step units in a runtime loop were 5% slower at B = 32).
// CAFXG_BLOCK=<B> forces a length (multiple of 8; 16..64 unrolled).
void pick_block(uint32_t max_iter, int precision, MandelLaunchCfg& c) {
  static const int env = [] {
    const char* e = getenv("CAFXG_BLOCK");
    return e ? atoi(e) : 0;
  }();
  auto set = [&](uint32_t b) {
    if (b >= 16 && b <= 64 && b % 8 == 0) {
      c.unit = (int)b;
      c.reps = 1;
    } else {
      c.unit = 8;
      c.reps = (int)(b / 8);
    }
  };
  if (env >= 8 && env % 8 == 0) {
    set((uint32_t)env);
    return;
  }
  const double alpha = precision ? 2.0 : 7.0, gamma = 0.002;
  uint32_t best = 32;
  double best_cost = 1e300;
  for (uint32_t b = 16; b <= 64; b += 8) {
    const double over = (double)((max_iter + b - 1) / b * b) / max_iter;
    const double cost = over * (1.0 + alpha / b) + gamma * b;
    if (cost < best_cost) {
      best = b;
      best_cost = cost;
    }
  }
  set(best);
}

MandelLaunchCfg mandel_cfg(Device* d, int precision, uint32_t max_iter,
                                  bool exact, bool safe, uint64_t pixels,
                                  const cafxg_tuning* tune) {
  MandelLaunchCfg c;
  // checked kernel: steps between votes (cfg1, max_iter 100: 16 steps 0.065 ms, 4 steps 0.074)
  c.ksteps = max_iter >= 512 ? 32 : max_iter >= 64 ? 16 : 4;
  static const int ks_env = [] {  // CAFXG_KSTEPS=4|16|32: experiments only
    const char* e = getenv("CAFXG_KSTEPS");
    return e ? atoi(e) : 0;
  }();
  if (ks_env == 4 || ks_env == 16 || ks_env == 32)
    c.ksteps = ks_env;
  c.exact = exact;
  static const uint32_t def_min = [] {  // CAFXG_DEFERRED_MIN=<max_iter>: experiments only
    const char* e = getenv("CAFXG_DEFERRED_MIN");
    return e ? (uint32_t)atoi(e) : 256u;
  }();
  c.deferred = safe && max_iter >= def_min && deferred_enabled();
  if (c.deferred) {
    pick_block(max_iter, precision, c);
    if (tune && tune->block_steps) {  // spawn_cl tuning (validated at spawn)
      c.unit = (int)tune->block_steps;
      c.reps = 1;
    }
  }
  // occupancy per kernel variant: [precision][checked ksteps 4/16/32 |
  // deferred unit 8/32][exact][deferred]
  const int vi = c.deferred ? c.unit / 8 - 1 : (c.ksteps == 4 ? 0 : c.ksteps == 16 ? 1 : 2);
  int& occ = d->mandel_occ[precision][vi][exact][c.deferred];
  if (occ == 0)
    occ = std::max(1, mandel_max_blocks_per_sm(precision, c.ksteps, exact, c.deferred,
                                               c.unit));
  const uint64_t per_block = (uint64_t)kMandelThreads * mandel_slots_per_thread(precision);
  uint64_t want = (pixels + per_block - 1) / per_block;
  uint64_t full = (uint64_t)d->sms * occ;
  c.grid = (int)std::max<uint64_t>(1, std::min(want, full));
  if (tune && tune->max_ctas)
    c.grid = std::min(c.grid, (int)tune->max_ctas);
  static const int occ_env = [] {  // CAFXG_OCC=<CTAs per SM>: experiments only
    const char* e = getenv("CAFXG_OCC");
    return e ? atoi(e) : 0;
  }();
  if (occ_env > 0)
    c.grid = std::min(c.grid, d->sms * occ_env);
  return c;
}

// Enqueues the Mandelbrot launches for `tiles` (all the same precision) on
// `stream`: one coordinate-table launch, then one escape launch per distinct
// max_iter (the kernel keeps max_iter launch-uniform). Descriptors beyond the
// inline capacity are uploaded first.
int launch_mandel_group(cafxg_ctx* ctx, Device* d, uint32_t* out_base,
                               std::vector<MTile>& tiles, int precision, bool exact,
                               cudaStream_t stream, bool coords_only, bool skip_coords,
                               uint32_t* direct_counters = nullptr,
                               const cafxg_tuning* tune = nullptr);

int launch_mandel(cafxg_ctx* ctx, Device* d, uint32_t* out_base,
                         const std::vector<MTile>& tiles_in, uint32_t total_chunks,
                         int precision, uint32_t max_iter, bool exact,
                         uint64_t pixels, cudaStream_t stream,
                         uint32_t* direct_counters, const cafxg_tuning* tune) {
  (void)max_iter;
  if (total_chunks == 0)
    return CAFXG_OK;
  // coordinate tables (one column and one row table per tile) pay off for
  // big tiles; batches of small tiles (request storms) compute coordinates
  // inline in the escape kernel and save the table launch
  std::vector<MTile> tiles = tiles_in;
  // (and so do launches of few pixels in all: kInlineCoordsPx)
  bool small_tiles = true;
  for (auto& t : tiles)
    small_tiles = small_tiles && (uint64_t)t.ncols * t.nrows <= (64u << 10);
  const bool small = small_tiles || pixels <= kInlineCoordsPx;
  uint8_t* coords = nullptr;
  if (!small) {
    const size_t esz = precision ? sizeof(double) : sizeof(float);
    uint64_t ncoord = 0;
    for (auto& t : tiles)
      ncoord += (uint64_t)t.ncols + t.nrows;
    CAFXG_CUDA_TRY(cudaMallocAsync((void**)&coords, ncoord * esz + 16, stream));
    uint64_t off = 0;
    for (auto& t : tiles) {
      t.cx = coords + off * esz;
      t.cy = coords + (off + t.ncols) * esz;
      off += (uint64_t)t.ncols + t.nrows;
    }
    CAFXG_TRY(
        launch_mandel_group(ctx, d, out_base, tiles, precision, exact, stream, true, false));
  } else {
    for (auto& t : tiles)
      t.cx = t.cy = nullptr;
  }
  // group by max_iter (stable), re-basing the chunk numbering per group
  std::vector<uint32_t> its;
  for (auto& t : tiles)
    if (std::find(its.begin(), its.end(), t.max_iter) == its.end())
      its.push_back(t.max_iter);
  for (uint32_t it : its) {
    std::vector<MTile> grp;
    for (auto& t : tiles)
      if (t.max_iter == it)
        grp.push_back(t);
    if (direct_counters && its.size() != 1)
      return fail(CAFXG_E_CONFIG, "internal: direct reply across max_iter groups");
    CAFXG_TRY(launch_mandel_group(ctx, d, out_base, grp, precision, exact, stream, false, true,
                                  direct_counters, tune));
  }
  if (coords)
    CAFXG_CUDA_TRY(cudaFreeAsync(coords, stream));
  return CAFXG_OK;
}

int launch_mandel_group(cafxg_ctx* ctx, Device* d, uint32_t* out_base,
                               std::vector<MTile>& tiles, int precision, bool exact,
                               cudaStream_t stream, bool coords_only, bool skip_coords,
                               uint32_t* direct_counters, const cafxg_tuning* tune) {
  uint32_t chunks = 0, max_extent = 0;
  uint64_t pixels = 0;
  for (auto& t : tiles) {
    t.chunk_begin = chunks;
    chunks += tile_chunks(t.nrows, t.ncols, (uint32_t)precision);
    pixels += (uint64_t)t.nrows * t.ncols;
    max_extent = std::max(max_extent, t.ncols + t.nrows);
  }
  if (chunks == 0)
    return CAFXG_OK;
  MLaunch L{};
  L.n = (uint32_t)tiles.size();
  L.total_chunks = chunks;
  L.max_iter = tiles[0].max_iter;
  L.out = out_base;
  for (auto& t : tiles)  // (the checked build traps on stores past it)
    L.out_limit = std::max<uint64_t>(L.out_limit, (uint64_t)t.out_off + (uint64_t)t.nrows * t.ncols);
#ifdef CAFXG_DEVICE_CHECKS
  // CAFXG_DCHECK_SELFTEST=1: a limit the launch must overrun, so a test can
  // see the checks fire
  static const bool dcheck_selftest = getenv("CAFXG_DCHECK_SELFTEST") != nullptr;
  if (dcheck_selftest)
    L.out_limit = 1;
#endif
  L.zero = 0.0f;
  L.inline_coords = tiles[0].cx == nullptr;
  if (direct_counters) {
    // run_mandel_batch checked the same conditions and skips the reply copy
    if (tiles.size() > (size_t)kInlineTiles || !L.inline_coords)
      return fail(CAFXG_E_CONFIG, "internal: direct reply on an ineligible batch");
    L.direct = 1;
    L.tile_done = direct_counters;
  }
  MTile* dev_tiles = nullptr;
  if (tiles.size() <= (size_t)kInlineTiles) {
    for (size_t i = 0; i < tiles.size(); ++i)
      L.inl[i] = tiles[i];
  } else {
    size_t bytes = tiles.size() * sizeof(MTile);
    CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dev_tiles, bytes, stream));
    CAFXG_TRY(upload(d, dev_tiles, tiles.data(), bytes, stream));
    ctx->st_h2d += bytes;
    L.tiles = dev_tiles;
  }
  if (!skip_coords) {
    int e = mandel_coords_launch(L, precision, max_extent, stream);
    if (e != 0)
      return cuda_status((cudaError_t)e, "mandelbrot coordinate launch");
    ctx->st_launches++;
  }
  if (!coords_only) {
    bool safe = true;
    for (auto& t : tiles)
      safe = safe && deferred_safe(t);
    MandelLaunchCfg cfg = mandel_cfg(d, precision, L.max_iter, exact, safe, pixels, tune);
    // a scheduler slot of the ring, reused only after the launch that held it
    // kSchedSlots launches ago finished (launches on different streams --
    // user streams of cafxg_mandelbrot_device included -- may run at once)
    const uint32_t slot = d->sched_acquire(stream);
    L.sched = d->sched + 2 * slot;
    const auto l0 = std::chrono::steady_clock::now();
    int e = mandel_launch(L, precision, cfg, stream);
    d->sched_release(slot, stream);
    ctx->st_phase_ns[5] += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                               std::chrono::steady_clock::now() - l0)
                               .count();
    if (e != 0)
      return cuda_status((cudaError_t)e, "mandelbrot launch");
    ctx->st_launches++;
    mark_used(ctx, d);
  }
  if (dev_tiles)
    CAFXG_CUDA_TRY(cudaFreeAsync(dev_tiles, stream));
  return CAFXG_OK;
}

// Splits the request's tiles into row-band sub-tiles dealt cyclically to the
// devices (contiguous bands are load-imbalanced up to 1.15x).
std::vector<std::vector<SubTile>> plan_mandel(
    const cafxg_mandel_desc* tiles, size_t n, size_t ndev) {
  std::vector<std::vector<SubTile>> per(ndev);
  uint64_t total = 0;
  for (size_t i = 0; i < n; ++i)
    total += (uint64_t)tiles[i].nrows * tiles[i].ncols;
  // band size: ~1M pixels when the request is large enough to share; a
  // single-device request of 1M..64M pixels goes in ~8 bands of >= 512K (four
  // for cfg1's 2M pixels), so copy-outs overlap the later bands' kernels
  // (a rank's 1/8 share of cfg3 is 32M pixels)
  static const uint64_t band_min = [] {  // CAFXG_BAND_MIN_KPX: experiments only
    const char* e = getenv("CAFXG_BAND_MIN_KPX");
    const int v = e ? atoi(e) : 0;
    return (v > 0 ? (uint64_t)v : 512ull) << 10;
  }();
  // Several devices: ~16 bands per device, 64K..1M pixels each, so cyclic
  // dealing balances the work and a request of a few M pixels still reaches
  // every device (cfg3 on 8 devices: 1M-pixel bands, 32 per device).
  const uint64_t band_px =
      ndev > 1 ? std::clamp<uint64_t>(total / (ndev * 16), 64ull << 10, 1ull << 20)
      : total > (64ull << 20) ? (1ull << 20)
      : total >= (1ull << 20) ? std::max<uint64_t>((total + 7) / 8, band_min)
                              : UINT64_MAX;
  size_t next = 0;
  for (size_t i = 0; i < n; ++i) {
    const cafxg_mandel_desc& t = tiles[i];
    uint64_t px = (uint64_t)t.nrows * t.ncols;
    if (px == 0)
      continue;
    uint32_t rows_per = band_px == UINT64_MAX
                            ? t.nrows
                            : (uint32_t)std::max<uint64_t>(1, band_px / t.ncols);
    for (uint32_t r = 0; r < t.nrows; r += rows_per) {
      SubTile s;
      s.d = t;
      s.d.row0 = t.row0 + r;
      s.d.nrows = std::min(rows_per, t.nrows - r);
      s.d.out_offset = t.out_offset + (uint64_t)r * t.ncols;
      s.pixels = (uint64_t)s.d.nrows * s.d.ncols;
      per[next % ndev].push_back(s);
      ++next;
    }
  }
  return per;
}

int stream_after(cudaStream_t b, cudaStream_t a);  // b waits for a's work so far
int stream_after_pooled(Device* d, cudaStream_t b, cudaStream_t a);

// Submits one device's share: waves of sub-tiles, each a single launch into a
// device staging buffer followed by the copy-out on the d2h stream, so the
// PCIe transfer of wave w overlaps the compute of wave w+1.
int submit_mandel_device(cafxg_ctx* ctx, Device* d,
                                const std::vector<SubTile>& subs,
                                uint32_t* host_out, bool out_pinned,
                                bool exact, Join* join, const cafxg_tuning* tune) {
  NvtxRange nvtx_range("cafxg.mandelbrot.device_share");
  cudaSetDevice(d->ordinal);
  std::lock_guard<std::mutex> g(d->submit_mu);
  static const uint64_t wave_px = [] {  // CAFXG_WAVE_MPX: experiments only
    const char* e = getenv("CAFXG_WAVE_MPX");
    const int v = e ? atoi(e) : 0;
    return (v > 0 ? (uint64_t)v : 32ull) << 20;
  }();
  uint32_t* staging = nullptr;  // pinned bounce buffer for pageable outputs
  uint64_t dev_px_total = 0;
  for (auto& s : subs)
    dev_px_total += s.pixels;
  if (!out_pinned) {
    staging = (uint32_t*)ctx->pinned.alloc(dev_px_total * 4);
    if (!staging)
      return fail(CAFXG_E_CONFIG, "mandelbrot: pinned staging allocation failed");
  }
  uint64_t staged = 0;
  std::vector<std::array<uint64_t, 3>> scat;  // (staging off, host off, px)
  size_t i = 0;
  // pixels still to schedule: waves shrink geometrically towards the end so
  // the copy-out left exposed after the last kernel is small
  uint64_t left = dev_px_total;
  // smallest wave: 2M pixels (launch overhead), 512K for small requests
  static const uint64_t big_min = [] {  // CAFXG_MIN_WAVE_MPX: experiments only
    const char* e = getenv("CAFXG_MIN_WAVE_MPX");
    const int v = e ? atoi(e) : 0;
    return (v > 0 ? (uint64_t)v : 2ull) << 20;
  }();
  static const uint64_t small_min = [] {  // CAFXG_SMALL_WAVE_KPX: experiments only
    const char* e = getenv("CAFXG_SMALL_WAVE_KPX");
    const int v = e ? atoi(e) : 0;
    return (v > 0 ? (uint64_t)v : 512ull) << 10;
  }();
  const uint64_t min_wave = dev_px_total >= (64ull << 20) ? big_min : small_min;
  // Small, shallow requests (<= 4M pixels, max_iter <= 256: cfg1) are bound by
  // the copy-out, not the kernel: one small first wave starts the copy engine
  // early and everything else goes in a second wave whose contiguous bands
  // leave in one copy (2 MB copies ran at ~45 GB/s, the link does ~55).
  // CAFXG_SMALL_PLAN=0: the geometric waves everywhere (experiments).
  static const bool small_plan_on = [] {
    const char* e = getenv("CAFXG_SMALL_PLAN");
    return !(e && e[0] == '0');
  }();
  uint32_t req_maxit = 0;
  for (auto& sb : subs)
    req_maxit = std::max(req_maxit, sb.d.max_iter);
  const bool two_waves = small_plan_on && dev_px_total <= (4ull << 20) && req_maxit <= 256;
  // CAFXG_TRACE=1: per-wave device timeline on stderr (debug aid)
  static const bool trace = [] {
    const char* e = getenv("CAFXG_TRACE");
    return e && e[0] == '1';
  }();
  std::vector<std::array<cudaEvent_t, 3>> tev;
  std::vector<double> thost;  // host clock at each wave's start / after its launches
  const double t_entry = trace_now_ms();
  // waves alternate between the two compute streams (both ordered after the
  // device's earlier work; compute is ordered after both at the end)
  uint32_t* dout_live = nullptr;  // the current wave's buffer until its free is queued
  // the waves; a failure part-way leaves earlier waves' copies queued, so it
  // is reported through the completion thread behind them (below)
  auto issue_waves = [&]() -> int {
    CAFXG_TRY(stream_after(d->compute2, d->compute));
    uint32_t wave = 0;
    while (i < subs.size()) {
      // (the two-wave plan keeps one stream: the first wave then runs alone and
      // its copy starts sooner)
      cudaStream_t ks = ((wave++ & 1) && !two_waves) ? d->compute2 : d->compute;
      // group a wave (same precision)
      size_t j = i;
      uint64_t px = 0;
      int prec = subs[i].d.precision;
      const uint64_t cap =
          two_waves ? (wave == 1 ? min_wave : UINT64_MAX)
                    : std::max<uint64_t>(std::min<uint64_t>(wave_px, left / 4), min_wave);
      while (j < subs.size() && subs[j].d.precision == prec &&
             (px == 0 || px + subs[j].pixels <= cap)) {
        px += subs[j].pixels;
        ++j;
      }
      uint32_t* dout = nullptr;
      CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dout, px * 4, ks));
      dout_live = dout;
      // CAFXG_FAIL_WAVE=<w>: wave w fails after its buffer exists (tests the
      // part-way failure path; never set in production)
      static const int fail_wave = [] {
        const char* e = getenv("CAFXG_FAIL_WAVE");
        return e ? atoi(e) : -1;
      }();
      if ((int)wave - 1 == fail_wave)
        return fail(CAFXG_E_DOWN, "mandelbrot: injected failure of wave %d", fail_wave);
      std::vector<MTile> mt(j - i);
      uint32_t chunks = 0, maxit = 0;
      uint64_t off = 0;
      for (size_t k = i; k < j; ++k) {
        fill_mtile(mt[k - i], subs[k].d, off, chunks);
        chunks += tile_chunks(subs[k].d.nrows, subs[k].d.ncols, subs[k].d.precision);
        maxit = std::max(maxit, subs[k].d.max_iter);
        off += subs[k].pixels;
      }
      if (trace) {
        tev.push_back({});
        for (auto& e : tev.back())
          cudaEventCreate(&e);
        cudaEventRecord(tev.back()[0], ks);
        thost.push_back(trace_now_ms());
      }
      CAFXG_TRY(launch_mandel(ctx, d, dout, mt, chunks, prec, maxit, exact, px, ks, nullptr,
                              tune));
      if (trace)
        thost.push_back(trace_now_ms());
      if (trace)
        cudaEventRecord(tev.back()[1], ks);
      CAFXG_TRY(stream_after_pooled(d, d->d2h, ks));
      off = 0;
      // copies of consecutive sub-tiles that are contiguous on both sides
      // (row bands of one tile into a pinned image; any run into the staging
      // buffer) go out as one cudaMemcpyAsync
      uint32_t* run_dst = nullptr;
      uint64_t run_src = 0, run_px = 0;
      auto flush_run = [&]() -> int {
        if (run_px) {
          CAFXG_CUDA_TRY(cudaMemcpyAsync(run_dst, dout + run_src, run_px * 4,
                                         cudaMemcpyDeviceToHost, d->d2h));
          ctx->st_d2h += run_px * 4;
        }
        run_px = 0;
        return CAFXG_OK;
      };
      for (size_t k = i; k < j; ++k) {
        uint32_t* dst;
        if (out_pinned) {
          dst = host_out + subs[k].d.out_offset;
        } else {
          dst = staging + staged;
          scat.push_back({staged, subs[k].d.out_offset, subs[k].pixels});
          staged += subs[k].pixels;
        }
        if (run_px && dst != run_dst + run_px)
          CAFXG_TRY(flush_run());
        if (!run_px) {
          run_dst = dst;
          run_src = off;
        }
        run_px += subs[k].pixels;
        off += subs[k].pixels;
      }
      CAFXG_TRY(flush_run());
      dout_live = nullptr;
      CAFXG_CUDA_TRY(cudaFreeAsync(dout, d->d2h));
      if (trace)
        cudaEventRecord(tev.back()[2], d->d2h);
      left -= px;
      i = j;
    }
    CAFXG_TRY(stream_after(d->compute, d->compute2));
    return CAFXG_OK;
  };
  const int issued = issue_waves();
  if (issued != CAFXG_OK) {
    // the caller's buffer may still be the target of queued
    // copies, so `done` must not fire before they drain. The copy stream is
    // ordered after both compute streams (best effort: on a dead device these
    // fail too, and the completion thread then sees the error), the live wave
    // buffer is freed there, and the staging buffer in the completion.
    std::string err = t_last_error;
    stream_after(d->d2h, d->compute);
    stream_after(d->d2h, d->compute2);
    if (dout_live)
      cudaFreeAsync(dout_live, d->d2h);
    cudaGetLastError();
    push_completion(ctx, d, d->d2h, [ctx, staging, join, issued, err](int) {
      if (staging)
        ctx->pinned.free(staging);
      set_last_error("%s", err.c_str());
      join->part_done(issued);
    });
    return CAFXG_OK;
  }
  if (trace && !tev.empty()) {
    cudaError_t se = cudaEventSynchronize(tev.back()[2]);
    for (size_t w = 0; w < tev.size(); ++w) {
      float a = -1, b = -1, c = -1;
      cudaError_t e1 = cudaEventElapsedTime(&a, tev[0][0], tev[w][0]);
      cudaError_t e2 = cudaEventElapsedTime(&b, tev[0][0], tev[w][1]);
      cudaError_t e3 = cudaEventElapsedTime(&c, tev[0][0], tev[w][2]);
      if (se || e1 || e2 || e3)
        fprintf(stderr, "cafxg trace errors %d %d %d %d\n", (int)se, (int)e1, (int)e2, (int)e3);
      fprintf(stderr, "cafxg trace wave %zu: kernel %.3f..%.3f ms, copy done %.3f ms\n", w, a, b,
              c);
    }
    for (size_t w = 0; w + 1 < thost.size(); w += 2)
      fprintf(stderr, "cafxg trace host: wave %zu issued %.3f..%.3f ms after entry\n", w / 2,
              thost[w] - t_entry, thost[w + 1] - t_entry);
    for (auto& w : tev)
      for (auto& e : w)
        cudaEventDestroy(e);
    cudaGetLastError();
  }
  push_completion(ctx, d, d->d2h,
                  [ctx, staging, scat = std::move(scat), host_out, join](int st) {
                    if (staging) {
                      if (st == CAFXG_OK)
                        for (auto& s : scat)
                          std::memcpy(host_out + s[1], staging + s[0], s[2] * 4);
                      ctx->pinned.free(staging);
                    }
                    join->part_done(st);
                  });
  return CAFXG_OK;
}

int mandel_submit_impl(cafxg_ctx* ctx, const cafxg_mandel_desc* tiles,
                              size_t n, uint32_t* host_out, cafxg_done_fn done,
                              void* user, const cafxg_tuning* tune) {
  NvtxRange nvtx_range("cafxg.mandelbrot.submit");
  if (!ctx || (n && !tiles) || (n && !host_out))
    return fail(CAFXG_E_CONFIG, "mandelbrot_submit: null argument");
  CAFXG_TRY(check_alive(ctx));
  uint64_t out_elems = 0;
  bool exact = false;
  for (size_t i = 0; i < n; ++i) {
    CAFXG_TRY(validate_mandel(tiles[i]));
    out_elems = std::max<uint64_t>(
        out_elems, tiles[i].out_offset + (uint64_t)tiles[i].nrows * tiles[i].ncols);
    exact = exact || use_exact(ctx, tiles[i]);
  }
  bool pinned = host_is_pinned(host_out, out_elems * 4);
  auto plan = plan_mandel(tiles, n, ctx->devs.size());
  Join* join = new Join;
  join->done = done;
  join->user = user;
  int parts = 0;
  for (auto& p : plan)
    parts += !p.empty();
  if (parts == 0) {
    // nothing to compute: complete through device 0's completion thread so
    // the callback still runs off the caller's thread
    join->remaining = 1;
    Device* d = ctx->devs[0].get();
    cudaSetDevice(d->ordinal);
    std::lock_guard<std::mutex> g(d->submit_mu);
    push_completion(ctx, d, d->compute, [join](int st) { join->part_done(st); });
    return CAFXG_OK;
  }
  join->remaining = parts;
  ctx->st_requests++;
  if (parts > 1) {
    // every device's share on its own issuer thread, all at once; a share
    // that fails before queueing anything reports through the join itself
    const bool tuned = tune != nullptr;
    const cafxg_tuning tcopy = tuned ? *tune : cafxg_tuning{};
    for (size_t k = 0; k < plan.size(); ++k) {
      if (plan[k].empty())
        continue;
      Device* d = ctx->devs[k].get();
      issue_async(ctx, d, [ctx, d, subs = std::move(plan[k]), host_out, pinned, exact, join, tuned,
                      tcopy] {
        const int s = submit_mandel_device(ctx, d, subs, host_out, pinned, exact, join,
                                           tuned ? &tcopy : nullptr);
        if (s != CAFXG_OK)
          join->part_done(s);
      });
    }
    return CAFXG_OK;
  }
  for (size_t k = 0; k < plan.size(); ++k) {
    if (plan[k].empty())
      continue;
    int s = submit_mandel_device(ctx, ctx->devs[k].get(), plan[k], host_out,
                                 pinned, exact, join, tune);
    if (s != CAFXG_OK) {
      // parts already submitted still report through the join
      std::string err = t_last_error;
      join->part_done(s);
      for (size_t r = k + 1; r < plan.size(); ++r)
        if (!plan[r].empty())
          join->part_done(s);
      t_last_error = err;
      return CAFXG_OK;  // the error is delivered through `done`
    }
  }
  return CAFXG_OK;
}

}  // namespace cafxg

using namespace cafxg;

extern "C" {

int cafxg_mandelbrot_submit(cafxg_ctx* ctx, const cafxg_mandel_desc* tiles, size_t n,
                            uint32_t* host_out, cafxg_done_fn done, void* user) {
  try {
    return mandel_submit_impl(ctx, tiles, n, host_out, done, user);
  } catch (const std::exception& ex) {
    return fail(CAFXG_E_CONFIG, "mandelbrot_submit: %s", ex.what());
  }
}

int cafxg_mandelbrot(cafxg_ctx* ctx, const cafxg_mandel_desc* tiles, size_t n,
                     uint32_t* host_out) try {
  Waiter w;
  int s = cafxg_mandelbrot_submit(ctx, tiles, n, host_out, &Waiter::cb, &w);
  if (s != CAFXG_OK)
    return s;
  return w.wait();
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_mandelbrot: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_mandelbrot: unknown exception");
}

int cafxg_mandelbrot_device(cafxg_ctx* ctx, int device, const cafxg_mandel_desc* tiles,
                            size_t n, uint32_t* dev_out, void* stream) {
  if (!ctx || device < 0 || device >= (int)ctx->devs.size() || (n && (!tiles || !dev_out)))
    return fail(CAFXG_E_CONFIG, "mandelbrot_device: bad argument");
  CAFXG_TRY(check_alive(ctx));
  try {
    Device* d = ctx->devs[device].get();
    bool exact = false;
    std::vector<MTile> mt;
    mt.reserve(n);
    uint32_t chunks = 0, maxit = 0;
    uint64_t px = 0, lo = UINT64_MAX, hi = 0;
    int prec = n ? (int)tiles[0].precision : 0;
    for (size_t i = 0; i < n; ++i) {
      CAFXG_TRY(validate_mandel(tiles[i]));
      if ((int)tiles[i].precision != prec)
        return fail(CAFXG_E_CONFIG, "mandelbrot_device: mixed precisions in one launch");
      uint64_t tp = (uint64_t)tiles[i].nrows * tiles[i].ncols;
      if (tp == 0)
        continue;  // empty tiles own no chunks
      lo = std::min<uint64_t>(lo, tiles[i].out_offset);
      hi = std::max<uint64_t>(hi, tiles[i].out_offset + tp);
    }
    if (hi > lo && hi - lo >= (1ull << 32))
      return fail(CAFXG_E_OUT_OF_RANGE, "mandelbrot_device: one launch spans >= 2^32 counts");
    for (size_t i = 0; i < n; ++i) {
      uint64_t tp = (uint64_t)tiles[i].nrows * tiles[i].ncols;
      if (tp == 0)
        continue;
      exact = exact || use_exact(ctx, tiles[i]);
      MTile m;
      fill_mtile(m, tiles[i], tiles[i].out_offset - lo, chunks);
      mt.push_back(m);
      chunks += tile_chunks(tiles[i].nrows, tiles[i].ncols, tiles[i].precision);
      maxit = std::max(maxit, tiles[i].max_iter);
      px += tp;
    }
    if (mt.empty())
      return CAFXG_OK;
    cudaSetDevice(d->ordinal);
    cudaStream_t s = stream ? (cudaStream_t)stream : d->compute;
    return launch_mandel(ctx, d, dev_out + lo, mt, chunks, prec, maxit, exact, px, s);
  } catch (const std::exception& ex) {
    return fail(CAFXG_E_CONFIG, "mandelbrot_device: %s", ex.what());
  }
}

int cafxg_fnv1a_u32_device(cafxg_ctx* ctx, int device, const uint32_t* cells, uint64_t n,
                           uint64_t seed, uint64_t* hash, void* stream) try {
  if (!ctx || !hash || device < 0 || device >= (int)ctx->devs.size() || (n && !cells))
    return fail(CAFXG_E_CONFIG, "fnv1a_u32_device: bad argument");
  Device* d = ctx->devs[device].get();
  cudaSetDevice(d->ordinal);
  cudaStream_t s = stream ? (cudaStream_t)stream : d->compute;
  void* scratch = nullptr;
  uint64_t* dhash = nullptr;
  CAFXG_CUDA_TRY(cudaMallocAsync(&scratch, fnv_scratch_bytes(n, d->sms), s));
  CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dhash, sizeof(uint64_t), s));
  int launches = 0;
  int e = fnv_launch(cells, n, seed, dhash, scratch, d->sms, s, &launches);
  if (e != 0)
    return cuda_status((cudaError_t)e, "fnv launch");
  ctx->st_launches += launches;
  CAFXG_CUDA_TRY(cudaMemcpyAsync(hash, dhash, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  CAFXG_CUDA_TRY(cudaFreeAsync(scratch, s));
  CAFXG_CUDA_TRY(cudaFreeAsync(dhash, s));
  CAFXG_CUDA_TRY(cudaStreamSynchronize(s));
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_fnv1a_u32_device: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_fnv1a_u32_device: unknown exception");
}

// run_mandelbrot(size, max_iter) (bench.cpp:481-505) on the context's devices:
// the reference-mode image (fp64, corner sampling, [-1.5,0.5]x[-1,1]) is
// computed in HBM in contiguous row blocks per device, each device hashes its
// block with the segment-table FNV (fnv.cu), and the per-device hashes are
// chained on the host in row order: the checksum is the reference's
// collector hash (bench.cpp:329-331) without moving the image off the GPUs.
int cafxg_run_mandelbrot(cafxg_ctx* ctx, uint32_t size, uint32_t max_iter, uint64_t* checksum,
                         double* wall_ms) try {
  NvtxRange nvtx_range("cafxg.run_mandelbrot");
  if (!ctx || !checksum || size == 0)
    return fail(CAFXG_E_CONFIG, "run_mandelbrot: bad argument");
  auto t0 = std::chrono::steady_clock::now();
  const size_t G = std::min<size_t>(ctx->devs.size(), size);
  std::vector<uint32_t*> img(G, nullptr);
  std::vector<uint64_t*> dh(G, nullptr);
  std::vector<uint64_t> hh(G, 0);
  std::vector<uint32_t> r0(G + 1);
  for (size_t g = 0; g <= G; ++g)
    r0[g] = (uint32_t)((uint64_t)size * g / G);
  // Per device: its block of rows in one escape launch, then the seed-
  // independent FNV pass 1 (per-segment low-byte tables, the bulk of the
  // hash) -- in parallel on every device. Then the cheap seeded passes run
  // device after device, each block seeded with the previous block's hash
  // (FNV is sequential). Overlapping pass 1 with the image on one device
  // was tried and is slower.
  std::vector<void*> scratch(G, nullptr);
  for (size_t g = 0; g < G; ++g) {
    Device* d = ctx->devs[g].get();
    cudaSetDevice(d->ordinal);
    uint64_t rows = r0[g + 1] - r0[g];
    uint64_t n = rows * size;
    CAFXG_CUDA_TRY(cudaMallocAsync((void**)&img[g], n * 4 + 16, d->compute));
    CAFXG_CUDA_TRY(cudaMallocAsync((void**)&dh[g], 8, d->compute));
    CAFXG_CUDA_TRY(cudaMallocAsync(&scratch[g], fnv_scratch_bytes(n, d->sms), d->compute));
    cafxg_mandel_desc t{};
    t.x0 = -1.5; t.x1 = 0.5; t.y0 = -1.0; t.y1 = 1.0;
    t.width = t.height = size;
    t.row0 = r0[g];
    t.nrows = (uint32_t)rows;
    t.ncols = size;
    t.max_iter = max_iter;
    t.precision = CAFXG_FP64;
    t.sampling = CAFXG_CORNER;
    CAFXG_TRY(validate_mandel(t));
    MTile m;
    fill_mtile(m, t, 0, 0);
    CAFXG_TRY(launch_mandel(ctx, d, img[g], {m}, tile_chunks(t.nrows, t.ncols, CAFXG_FP64), CAFXG_FP64,
                            max_iter, use_exact(ctx, t), n, d->compute));
    uint64_t seg_cells = 0;
    uint32_t nseg = 0;
    fnv_segments(n, d->sms, &seg_cells, &nseg);
    int e = fnv_lowbyte_launch(img[g], n, 0, nseg, scratch[g], d->sms, d->compute);
    if (e != 0)
      return cuda_status((cudaError_t)e, "fnv pass-1 launch");
    ctx->st_launches++;
  }
  // the seeded passes, block after block
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t g = 0; g < G; ++g) {
    Device* d = ctx->devs[g].get();
    cudaSetDevice(d->ordinal);
    uint64_t n = (uint64_t)(r0[g + 1] - r0[g]) * size;
    int launches = 0;
    int e = fnv_finish_launch(img[g], n, h, dh[g], scratch[g], d->sms, d->compute, &launches);
    if (e != 0)
      return cuda_status((cudaError_t)e, "fnv launch");
    ctx->st_launches += launches;
    CAFXG_CUDA_TRY(cudaMemcpyAsync(&hh[g], dh[g], 8, cudaMemcpyDeviceToHost, d->compute));
    CAFXG_CUDA_TRY(cudaStreamSynchronize(d->compute));
    h = hh[g];
  }
  for (size_t g = 0; g < G; ++g) {
    Device* d = ctx->devs[g].get();
    cudaSetDevice(d->ordinal);
    cudaFreeAsync(img[g], d->compute);
    cudaFreeAsync(dh[g], d->compute);
    cudaFreeAsync(scratch[g], d->compute);
  }
  *checksum = h;
  if (wall_ms)
    *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                   .count();
  return CAFXG_OK;
} catch (const std::exception& ex) {
  return fail(CAFXG_E_CONFIG, "cafxg_run_mandelbrot: %s", ex.what());
} catch (...) {
  return fail(CAFXG_E_CONFIG, "cafxg_run_mandelbrot: unknown exception");
}

}  // extern "C"
