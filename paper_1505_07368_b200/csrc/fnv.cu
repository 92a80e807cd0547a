// FNV-1a-64 of a u32 array hashed as big-endian bytes (cafx::detail::
// fnv1a_u32, /root/reference/proj/include/cafx/detail/fnv.hpp:23-28) -- the
// run_mandelbrot checksum (bench.cpp:329-331) -- computed on the device.
//
// FNV-1a is a sequential byte recurrence h' = (h ^ b) * p (mod 2^64), so it
// is parallelised through a decomposition of the state rather than of the
// data. Write h = 256u + l with l the low byte. Because b < 256 and p is odd,
//     (256u + (l ^ b)) * p = 256 (u*p + q) + r,   t = l ^ b, t*p = 256q + r,
// so the low byte evolves on its own, l' = (t * 179) mod 256 (435 = 179 mod
// 256; a permutation of 0..255), and the high part is affine in u with slope
// p: u' = u*p + q(l, b), q = (t << 32) + (t*435 >> 8) (p = 2^40 + 435).
//
// Three passes:
//  1. low bytes only. A segment's 256 possible incoming low bytes are
//     tracked at once by one warp, two per 32-bit register (16-bit slots:
//     one LOP3 + one IMAD advance two lanes by a byte), and recorded at
//     every sub-segment boundary;
//  2. one thread walks the segments' low-byte permutations from the seed,
//     giving each segment its real incoming low byte;
//  3. one thread per sub-segment runs the full recurrence from its real
//     incoming low byte (read from the pass-1 record); each warp composes its
//     32 affine maps into the segment's, and a final thread folds the
//     segments in order.
// All passes are parallel except two short sequential walks over the
// segments; the result is bit-identical to the serial loop.
#include <cuda_runtime.h>

#include <cstdint>

namespace cafxg {
namespace {

constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr int kP1Threads = 32;   // one warp per segment: 32 threads x 8 low bytes
constexpr int kSubSegs = 32;     // sub-segments per segment (pass 3: one warp)
constexpr int kTile = 256;       // cells staged in smem per round (pass 1; 4 KB, 32 warps/SM)
constexpr int kRecWords = 64;    // 256 low bytes = 64 packed words per record

// Pass 1: per segment, the low byte after every sub-segment for all 256
// incoming low bytes (128 tracked, see below), two per register in 16-bit
// slots (value in bits 0-7 / 16-23): one step is
// r = ((r ^ b) & 0x00ff00ff) * 179 -- one LOP3 and one IMAD per two lanes
// (179 * 255 < 2^16, so the slots never interfere; the next step's mask
// drops the product's high byte). rec[(seg * kSubSegs + j) * 64 + w] holds
// low bytes 4w..4w+3 at the START of sub-segment j; L[seg * 256 + v] is the
// outgoing low byte for incoming v.
__global__ void __launch_bounds__(kP1Threads)
    fnv_lowbyte_kernel(const uint32_t* __restrict__ cells, uint64_t n, uint64_t seg_cells,
                       uint64_t sub_cells, uint32_t* __restrict__ rec,
                       uint8_t* __restrict__ L, uint32_t seg0) {
  const uint32_t seg = seg0 + blockIdx.x;
  // each staged cell pre-expanded into its four steps' operands (byte b in
  // both 16-bit slots, big-endian order): the inner loop reads them with one
  // broadcast 16-byte load instead of a load and four byte permutes per lane
  __shared__ uint4 tile[kTile];
  const uint64_t begin = (uint64_t)seg * seg_cells;
  const uint64_t end = begin + seg_cells < n ? begin + seg_cells : n;
  const uint32_t tid = threadIdx.x;
  // Only incoming low bytes 0..127 are tracked: every step is "bit j flips
  // with input bit j, plus a function of the lower bits" (XOR with a byte,
  // multiplication by an odd constant), and so is any composition of steps;
  // hence out(v + 128) = out(v) ^ 128 and the other half of every record and
  // table is the tracked half with the top bit flipped. Lane t tracks values
  // 4t..4t+3 in two registers (two 16-bit slots each).
  uint32_t r[2];
#pragma unroll
  for (int k = 0; k < 2; ++k)
    r[k] = (4 * tid + 2 * k) | ((4 * tid + 2 * k + 1) << 16);
  uint32_t* myrec = rec + (size_t)seg * kSubSegs * kRecWords + tid;
  auto record = [&](uint32_t j) {
    // low bytes of the slots, packed in incoming-value order
    const uint32_t w = __byte_perm(r[0], r[1], 0x6420);
    myrec[(size_t)j * kRecWords] = w;
    myrec[(size_t)j * kRecWords + 32] = w ^ 0x80808080u;
  };
  auto step = [&](uint32_t bb) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      r[k] = ((r[k] ^ bb) & 0x00ff00ffu) * 179u;
  };
  uint64_t next_rec = begin;  // cell index of the next sub-segment start
  uint32_t j = 0;
  for (uint64_t base = begin; base < end; base += kTile) {
    const uint32_t cnt = end - base < (uint64_t)kTile ? (uint32_t)(end - base) : kTile;
    __syncwarp();
    for (uint32_t i = tid; i < cnt; i += kP1Threads) {
      const uint32_t x = __ldg(cells + base + i);
      tile[i] = make_uint4(__byte_perm(x, 0, 0x4343), __byte_perm(x, 0, 0x4242),
                           __byte_perm(x, 0, 0x4141), __byte_perm(x, 0, 0x4040));
    }
    __syncwarp();
    uint32_t i = 0;
    while (i < cnt) {
      // run to the next sub-segment start (or the tile end) without tests
      uint32_t stop = cnt;
      if (next_rec < base + cnt) {
        if (next_rec == base + i) {
          record(j);
          ++j;
          next_rec += sub_cells;
          continue;
        }
        stop = (uint32_t)(next_rec - base);
      }
#pragma unroll 4
      for (; i < stop; ++i) {
        const uint4 v = tile[i];  // broadcast read
        step(v.x);
        step(v.y);
        step(v.z);
        step(v.w);
      }
    }
  }
  for (; j < kSubSegs; ++j)  // empty trailing sub-segments start where we end
    record(j);
  uint32_t* out = reinterpret_cast<uint32_t*>(L + (size_t)seg * 256) + tid;
  const uint32_t w = __byte_perm(r[0], r[1], 0x6420);
  out[0] = w;
  out[32] = w ^ 0x80808080u;
}

// Pass 2: the real incoming low byte of every segment, and the final one.
// Segment maps compose, so the walk is two-level: (a) one warp per group of
// kGroup segments composes the group's tables into one; (b) one thread walks
// the group tables from the seed; (c) one thread per group walks its own
// segments from the group's incoming byte.
constexpr uint32_t kGroup = 64;

__global__ void __launch_bounds__(32)
    fnv_group_tables_kernel(const uint8_t* __restrict__ L, uint32_t nseg,
                            uint8_t* __restrict__ GT) {
  const uint32_t g = blockIdx.x, lane = threadIdx.x;
  const uint32_t s0 = g * kGroup, s1 = min(nseg, s0 + kGroup);
  uint32_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
    v[i] = lane * 8 + i;  // T = identity on the lane's 8 values
  for (uint32_t k = s0; k < s1; ++k) {
    const uint8_t* t = L + (size_t)k * 256;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      v[i] = __ldg(t + v[i]);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
    GT[(size_t)g * 256 + lane * 8 + i] = (uint8_t)v[i];
}

__global__ void fnv_group_walk_kernel(const uint8_t* __restrict__ GT, uint32_t ngroups,
                                      uint64_t seed, uint8_t* __restrict__ gin) {
  uint32_t l = (uint32_t)(seed & 255u);
  for (uint32_t g = 0; g < ngroups; ++g) {
    gin[g] = (uint8_t)l;
    l = GT[(size_t)g * 256 + l];
  }
  gin[ngroups] = (uint8_t)l;
}

__global__ void __launch_bounds__(256)
    fnv_segment_walk_kernel(const uint8_t* __restrict__ L, uint32_t nseg,
                            const uint8_t* __restrict__ gin, uint8_t* __restrict__ lin) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t ngroups = (nseg + kGroup - 1) / kGroup;
  if (g >= ngroups)
    return;
  uint32_t l = gin[g];
  const uint32_t s0 = g * kGroup, s1 = min(nseg, s0 + kGroup);
  for (uint32_t k = s0; k < s1; ++k) {
    lin[k] = (uint8_t)l;
    l = __ldg(L + (size_t)k * 256 + l);
  }
  if (s1 == nseg)
    lin[nseg] = (uint8_t)l;
}

__device__ __forceinline__ uint64_t pow_dev(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1)
      r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

// Pass 3: thread = (segment, sub-segment) -- a warp is one segment: full
// recurrence from the real incoming low byte gives the sub-segment's affine
// map u -> p^(4 len) u + c; the warp composes its 32 maps in order
// ((P1,C1) then (P2,C2) = (P1 P2, C1 P2 + C2)) and lane 0 stores the
// segment's (P, C).
__global__ void __launch_bounds__(256)
    fnv_affine_kernel(const uint32_t* __restrict__ cells, uint64_t n, uint64_t seg_cells,
                      uint64_t sub_cells, uint32_t nseg, const uint32_t* __restrict__ rec,
                      const uint8_t* __restrict__ lin, uint64_t* __restrict__ SP,
                      uint64_t* __restrict__ SC) {
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (uint64_t)nseg * kSubSegs)
    return;  // whole warps only: nseg * 32 threads
  const uint32_t s = (uint32_t)(g / kSubSegs), j = (uint32_t)(g % kSubSegs);
  const uint64_t seg_begin = (uint64_t)s * seg_cells;
  const uint64_t seg_end = seg_begin + seg_cells < n ? seg_begin + seg_cells : n;
  uint64_t b = seg_begin + (uint64_t)j * sub_cells;
  uint64_t e = b + sub_cells;
  if (b > seg_end) b = seg_end;
  if (e > seg_end) e = seg_end;
  const uint32_t v = lin[s];
  const uint32_t word = rec[((size_t)s * kSubSegs + j) * kRecWords + (v >> 2)];
  uint32_t l = (word >> (8 * (v & 3))) & 255u;
  uint64_t c = 0;
  for (uint64_t i = b; i < e; ++i) {
    const uint32_t x = __ldg(cells + i);
#pragma unroll
    for (int sh = 24; sh >= 0; sh -= 8) {
      const uint32_t t = l ^ ((x >> sh) & 255u);
      const uint32_t m = t * 435u;
      l = m & 255u;
      c = c * kFnvPrime + (((uint64_t)t << 32) + (m >> 8));
    }
  }
  uint64_t P = pow_dev(kFnvPrime, 4 * (e - b));
  const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint64_t P2 = __shfl_down_sync(0xffffffffu, P, off);
    const uint64_t C2 = __shfl_down_sync(0xffffffffu, c, off);
    if (lane + off < 32 && (lane & (2 * off - 1)) == 0) {
      c = c * P2 + C2;
      P = P * P2;
    }
  }
  if (lane == 0) {
    SP[s] = P;
    SC[s] = c;
  }
}

// Fold: u = u * P_s + C_s over the segments in order, two-level like the
// walk: one thread composes each group's maps ((P1,C1) then (P2,C2) =
// (P1 P2, C1 P2 + C2)), one thread folds the groups from the seed.
__global__ void __launch_bounds__(256)
    fnv_group_affine_kernel(const uint64_t* __restrict__ SP, const uint64_t* __restrict__ SC,
                            uint32_t nseg, uint64_t* __restrict__ GP,
                            uint64_t* __restrict__ GC) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t ngroups = (nseg + kGroup - 1) / kGroup;
  if (g >= ngroups)
    return;
  uint64_t P = 1, C = 0;
  const uint32_t s0 = g * kGroup, s1 = min(nseg, s0 + kGroup);
  for (uint32_t k = s0; k < s1; ++k) {
    const uint64_t p2 = SP[k];
    C = C * p2 + SC[k];
    P = P * p2;
  }
  GP[g] = P;
  GC[g] = C;
}

__global__ void fnv_fold_kernel(const uint64_t* __restrict__ GP, const uint64_t* __restrict__ GC,
                                uint32_t ngroups, uint64_t seed,
                                const uint8_t* __restrict__ last_low, uint64_t* out) {
  uint64_t u = seed >> 8;
  for (uint32_t g = 0; g < ngroups; ++g)
    u = u * GP[g] + GC[g];
  *out = (u << 8) | *last_low;
}

uint64_t pow_mod64(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1)
      r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

struct FnvPlan {
  uint64_t seg_cells, sub_cells;
  uint32_t nseg;
};

FnvPlan plan(uint64_t n, int sms) {
  FnvPlan p;
  uint64_t want = (uint64_t)sms * 32;  // pass-1 CTAs: 32 one-warp CTAs per SM
  p.seg_cells = (n + want - 1) / want;
  if (p.seg_cells < 4096)
    p.seg_cells = 4096;
  p.nseg = n ? (uint32_t)((n + p.seg_cells - 1) / p.seg_cells) : 0;
  p.sub_cells = (p.seg_cells + kSubSegs - 1) / kSubSegs;
  return p;
}

}  // namespace

size_t fnv_scratch_bytes(uint64_t n, int sms) {
  FnvPlan p = plan(n, sms);
  const size_t ng = (p.nseg + kGroup - 1) / kGroup;
  size_t rec = (size_t)p.nseg * kSubSegs * kRecWords * sizeof(uint32_t);
  size_t L = (size_t)p.nseg * 256;
  size_t PC = (size_t)p.nseg * 2 * sizeof(uint64_t);
  size_t groups = ng * 2 * sizeof(uint64_t) + ng * 256 + ng + 1;
  return PC + rec + L + p.nseg + 1 + groups + 256;
}

namespace {
struct FnvScratch {
  uint64_t *SP, *SC, *GP, *GC;
  uint32_t* rec;
  uint8_t *L, *lin, *GT, *gin;
  uint32_t ngroups;
};
FnvScratch carve(const FnvPlan& p, void* scratch) {
  FnvScratch x;
  x.ngroups = (p.nseg + kGroup - 1) / kGroup;
  x.SP = static_cast<uint64_t*>(scratch);
  x.SC = x.SP + p.nseg;
  x.GP = x.SC + p.nseg;
  x.GC = x.GP + x.ngroups;
  x.rec = reinterpret_cast<uint32_t*>(x.GC + x.ngroups);
  x.L = reinterpret_cast<uint8_t*>(x.rec + (size_t)p.nseg * kSubSegs * kRecWords);
  x.lin = x.L + (size_t)p.nseg * 256;
  x.GT = x.lin + p.nseg + 1;
  x.gin = x.GT + (size_t)x.ngroups * 256;
  return x;
}
}  // namespace

void fnv_segments(uint64_t n, int sms, uint64_t* seg_cells, uint32_t* nseg) {
  FnvPlan p = plan(n, sms);
  *seg_cells = p.seg_cells;
  *nseg = p.nseg;
}

int fnv_lowbyte_launch(const uint32_t* cells, uint64_t n, uint32_t seg_begin, uint32_t seg_count,
                       void* scratch, int sms, void* stream) {
  FnvPlan p = plan(n, sms);
  if (seg_begin >= p.nseg || seg_count == 0)
    return 0;
  if (seg_count > p.nseg - seg_begin)
    seg_count = p.nseg - seg_begin;
  FnvScratch x = carve(p, scratch);
  fnv_lowbyte_kernel<<<seg_count, kP1Threads, 0, (cudaStream_t)stream>>>(
      cells, n, p.seg_cells, p.sub_cells, x.rec, x.L, seg_begin);
  return (int)cudaGetLastError();
}

int fnv_finish_launch(const uint32_t* cells, uint64_t n, uint64_t seed, uint64_t* out,
                      void* scratch, int sms, void* stream, int* launches) {
  cudaStream_t st = (cudaStream_t)stream;
  FnvPlan p = plan(n, sms);
  FnvScratch x = carve(p, scratch);
  int k = 0;
  const uint32_t ng = x.ngroups;
  if (p.nseg) {
    fnv_group_tables_kernel<<<ng, 32, 0, st>>>(x.L, p.nseg, x.GT);
    fnv_group_walk_kernel<<<1, 1, 0, st>>>(x.GT, ng, seed, x.gin);
    fnv_segment_walk_kernel<<<(ng + 255) / 256, 256, 0, st>>>(x.L, p.nseg, x.gin, x.lin);
    uint64_t threads = (uint64_t)p.nseg * kSubSegs;
    fnv_affine_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
        cells, n, p.seg_cells, p.sub_cells, p.nseg, x.rec, x.lin, x.SP, x.SC);
    fnv_group_affine_kernel<<<(ng + 255) / 256, 256, 0, st>>>(x.SP, x.SC, p.nseg, x.GP, x.GC);
    k += 5;
  } else {
    cudaMemsetAsync(x.lin, (int)(seed & 255u), 1, st);  // no cells: low byte = seed's
  }
  fnv_fold_kernel<<<1, 1, 0, st>>>(x.GP, x.GC, ng, seed, x.lin + p.nseg, out);
  ++k;
  if (launches)
    *launches = k;
  return (int)cudaGetLastError();
}

// Enqueues the device FNV of `n` cells onto `stream`; the 64-bit hash lands
// in device memory `out`. Scratch: fnv_scratch_bytes(n, sms).
int fnv_launch(const uint32_t* cells, uint64_t n, uint64_t seed, uint64_t* out, void* scratch,
               int sms, void* stream, int* launches) {
  FnvPlan p = plan(n, sms);
  int e = fnv_lowbyte_launch(cells, n, 0, p.nseg, scratch, sms, stream);
  if (e)
    return e;
  int k = 0;
  e = fnv_finish_launch(cells, n, seed, out, scratch, sms, stream, &k);
  if (launches)
    *launches = k + (p.nseg ? 1 : 0);
  return e;
}

}  // namespace cafxg
