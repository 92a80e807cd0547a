// Kernel -> mapped pinned host write bandwidth (reply scatter design probe).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void scatter(const uint4* src, uint4* dst, size_t seg16, int nseg, int unroll) {
  for (int s = blockIdx.x; s < nseg; s += gridDim.x) {
    const uint4* a = src + (size_t)s * seg16;
    uint4* b = dst + (size_t)s * seg16;
    for (size_t i = threadIdx.x; i < seg16; i += blockDim.x)
      b[i] = a[i];
  }
}

int main() {
  const int nseg = 16384;
  const size_t seg = 16384;  // bytes
  uint4 *src, *dst;
  cudaMalloc(&src, nseg * seg);
  cudaHostAlloc((void**)&dst, nseg * seg, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {8, 16, 32, 48, 64, 148})
    for (int threads : {256, 512, 1024}) {
      scatter<<<grid, threads>>>(src, dst, seg / 16, nseg, 1);
      cudaEventRecord(a);
      scatter<<<grid, threads>>>(src, dst, seg / 16, nseg, 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("grid %5d threads %4d: %.2f ms  %.1f GB/s\n", grid, threads, ms, nseg * seg / ms / 1e6);
    }
  // reference: copy engine D2H of the same bytes
  cudaEventRecord(a);
  cudaMemcpyAsync(dst, src, nseg * seg, cudaMemcpyDeviceToHost);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("copy engine: %.2f ms %.1f GB/s\n", ms, nseg * seg / ms / 1e6);
  return 0;
}
