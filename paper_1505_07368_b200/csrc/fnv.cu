// FNV-1a-64 of a u32 array hashed as big-endian bytes (cafx::detail::
// fnv1a_u32, /root/reference/proj/include/cafx/detail/fnv.hpp:23-28) -- the
// run_mandelbrot checksum (bench.cpp:329-331) -- computed on the device.
//
// FNV-1a is a sequential byte recurrence h' = (h ^ b) * p (mod 2^64), so it
// is parallelised through a decomposition of the state rather than of the
// data. Write h = 256u + l with l the low byte. Because b < 256 and p is odd,
//     (256u + (l ^ b)) * p = 256 (u*p + q) + r,   t = l ^ b, t*p = 256q + r,
// so the low byte evolves on its own (l' = r, a permutation of 0..255) and the
// high part is affine in u with slope p: u' = u*p + q(l, b). A segment of n
// bytes therefore acts as
//     l_end = L[l0],   u_end = p^n * u0 + Cs[l0]   (mod 2^56; computed mod 2^64)
// for a 256-entry table pair (L, Cs). One CTA of 256 threads builds a
// segment's tables (thread = starting low byte); a single thread then walks
// the segments in order from the real seed. Work is 256x the serial hash but
// spread over the whole GPU, and the result is bit-identical to the
// reference's serial loop.
//
// With p = 2^40 + 435:  t*p = t*2^40 + t*435, so q = (t << 32) + (t*435 >> 8)
// and r = t*435 & 255 (t*435 < 2^17).
#include <cuda_runtime.h>

#include <cstdint>

namespace cafxg {
namespace {

constexpr uint64_t kFnvPrime = 0x100000001b3ull;
constexpr int kFnvThreads = 256;
constexpr int kFnvTile = 2048;  // cells staged in smem per round

__global__ void __launch_bounds__(kFnvThreads)
    fnv_segments_kernel(const uint32_t* __restrict__ cells, uint64_t n, uint64_t seg_cells,
                        uint8_t* __restrict__ Lout, uint64_t* __restrict__ Cout) {
  __shared__ uint32_t tile[kFnvTile];
  const uint64_t begin = (uint64_t)blockIdx.x * seg_cells;
  const uint64_t end = begin + seg_cells < n ? begin + seg_cells : n;
  uint32_t l = threadIdx.x;  // this thread's starting low byte
  uint64_t c = 0;
  for (uint64_t base = begin; base < end; base += kFnvTile) {
    const uint32_t cnt = end - base < (uint64_t)kFnvTile ? (uint32_t)(end - base) : kFnvTile;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += kFnvThreads)
      tile[i] = __ldg(cells + base + i);
    __syncthreads();
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t x = tile[i];  // broadcast read
#pragma unroll
      for (int sh = 24; sh >= 0; sh -= 8) {
        const uint32_t t = l ^ ((x >> sh) & 255u);
        const uint32_t m = t * 435u;
        l = m & 255u;
        c = c * kFnvPrime + (((uint64_t)t << 32) + (m >> 8));
      }
    }
  }
  Lout[(size_t)blockIdx.x * 256 + threadIdx.x] = (uint8_t)l;
  Cout[(size_t)blockIdx.x * 256 + threadIdx.x] = c;
}

// Walks the segment tables from the seed: one thread, nseg steps.
__global__ void fnv_walk_kernel(const uint8_t* __restrict__ L, const uint64_t* __restrict__ C,
                                uint64_t nseg, uint64_t p_full, uint64_t p_last,
                                uint64_t seed, uint64_t* out) {
  uint32_t l = (uint32_t)(seed & 255u);
  uint64_t u = seed >> 8;
  for (uint64_t s = 0; s < nseg; ++s) {
    const uint64_t pn = (s + 1 == nseg) ? p_last : p_full;
    u = u * pn + C[s * 256 + l];
    l = L[s * 256 + l];
  }
  *out = ((u << 8) | l);
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

}  // namespace

// Enqueues the device FNV of `n` cells onto `stream`; the 64-bit hash lands
// in device memory `out`. Scratch: fnv_scratch_bytes(n, sms).
uint64_t fnv_segment_cells(uint64_t n, int sms) {
  uint64_t want = (uint64_t)sms * 8;  // one wave of 8 CTAs per SM
  uint64_t seg = (n + want - 1) / want;
  return seg < 256 ? 256 : seg;
}

size_t fnv_scratch_bytes(uint64_t n, int sms) {
  uint64_t seg = fnv_segment_cells(n, sms);
  uint64_t nseg = n ? (n + seg - 1) / seg : 0;
  return nseg * 256 * (sizeof(uint64_t) + 1) + 16;
}

int fnv_launch(const uint32_t* cells, uint64_t n, uint64_t seed, uint64_t* out, void* scratch,
               int sms, void* stream, int* launches) {
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t seg = fnv_segment_cells(n, sms);
  uint64_t nseg = n ? (n + seg - 1) / seg : 0;
  uint64_t* C = static_cast<uint64_t*>(scratch);
  uint8_t* L = reinterpret_cast<uint8_t*>(C + nseg * 256);
  int k = 0;
  if (nseg) {
    fnv_segments_kernel<<<(unsigned)nseg, kFnvThreads, 0, s>>>(cells, n, seg, L, C);
    ++k;
  }
  uint64_t last = nseg ? n - (nseg - 1) * seg : 0;
  fnv_walk_kernel<<<1, 1, 0, s>>>(L, C, nseg, pow_mod64(kFnvPrime, 4 * seg),
                                  pow_mod64(kFnvPrime, 4 * last), seed, out);
  ++k;
  if (launches)
    *launches = k;
  return (int)cudaGetLastError();
}

}  // namespace cafxg
