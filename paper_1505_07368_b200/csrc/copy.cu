// Reply scatter: copies each request's counts from the batch's device staging
// buffer straight into its (mapped, pinned) host reply buffer, so a batch of
// N small replies costs one launch instead of N cudaMemcpyAsync calls.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "common.hpp"

namespace cafxg {
namespace {

__device__ __forceinline__ void copy_segment(const CopySeg& g) {
  const uintptr_t a = (uintptr_t)g.src | (uintptr_t)g.dst | (uintptr_t)g.bytes;
  if ((a & 15u) == 0) {
    const uint4* src = (const uint4*)g.src;
    uint4* dst = (uint4*)g.dst;
    const uint64_t n16 = g.bytes >> 4;
    for (uint64_t i = threadIdx.x; i < n16; i += blockDim.x)
      dst[i] = __ldg(src + i);
  } else {
    const uint8_t* src = (const uint8_t*)g.src;
    uint8_t* dst = (uint8_t*)g.dst;
    for (uint64_t i = threadIdx.x; i < g.bytes; i += blockDim.x)
      dst[i] = src[i];
  }
}

__global__ void __launch_bounds__(1024) copy_segments_kernel(const CopySeg* segs,
                                                            uint32_t n) {
  for (uint32_t s = blockIdx.x; s < n; s += gridDim.x)
    copy_segment(segs[s]);
}

struct InlineSegs {
  CopySeg s[kInlineSegs];
};

__global__ void __launch_bounds__(1024) copy_segments_inline_kernel(
    const __grid_constant__ InlineSegs segs, uint32_t n) {
  for (uint32_t s = blockIdx.x; s < n; s += gridDim.x)
    copy_segment(segs.s[s]);
}

}  // namespace

// CTAs of a scatter launch: a few wide CTAs already saturate PCIe writes and
// leave the other SMs to the next batch's escape kernel (CAFXG_SCATTER_CTAS
// overrides, experiments only)
static uint32_t scatter_ctas(uint32_t n) {
  static const uint32_t cap = [] {
    const char* e = getenv("CAFXG_SCATTER_CTAS");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? (uint32_t)v : 16u;
  }();
  return n < cap ? n : cap;
}

int copy_segments_inline_launch(const CopySeg* segs_host, uint32_t n, void* stream) {
  if (n == 0)
    return 0;
  if (n > kInlineSegs)
    return (int)cudaErrorInvalidValue;
  InlineSegs p;
  for (uint32_t i = 0; i < n; ++i)
    p.s[i] = segs_host[i];
  uint32_t grid = scatter_ctas(n);
  copy_segments_inline_kernel<<<grid, 1024, 0, (cudaStream_t)stream>>>(p, n);
  return (int)cudaGetLastError();
}

int copy_segments_launch(const CopySeg* segs_dev, uint32_t n, void* stream) {
  if (n == 0)
    return 0;
  // A few wide CTAs already saturate PCIe writes (~53 GB/s measured with
  // 16 x 1024 threads); leaving the other SMs free lets the next batch's
  // escape kernel run concurrently on the compute stream.
  uint32_t grid = scatter_ctas(n);
  copy_segments_kernel<<<grid, 1024, 0, (cudaStream_t)stream>>>(segs_dev, n);
  return (int)cudaGetLastError();
}

}  // namespace cafxg
