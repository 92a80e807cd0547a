// fp32 SIMT GEMM (FFMA, register-tiled): the correctness anchor of the
// `matrix_multiply` compute actor and the fallback for
// shapes the tcgen05 3xTF32 kernel does not take.
//
// C[M,N] = A[M,K] * B[K,N], row-major, fp32 accumulate.
// 128x128 block tile, BK = 16, 256 threads, 8x8 outputs per thread laid out
// as two 4x4 quadrants 64 apart (conflict-free float4 smem reads), register
// double buffering of the next K tile.
#include <cuda_runtime.h>

#include <cstdint>

#include "sgemm.cuh"

namespace cafxg {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, NT = 256;

template <bool kAligned>
__device__ __forceinline__ void load_a(const float* __restrict__ A, int lda,
                                       int M, int K, int m0, int k0,
                                       float (&ra)[8]) {
  // 128 rows x 16 k: thread t loads rows (t>>2) and (t>>2)+64, k = (t&3)*4..
  const int r = threadIdx.x >> 2, c = (threadIdx.x & 3) * 4;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int gm = m0 + r + h * 64, gk = k0 + c;
    if (kAligned && gm < M && gk + 3 < K) {
      float4 v = __ldg(reinterpret_cast<const float4*>(A + (size_t)gm * lda + gk));
      ra[h * 4 + 0] = v.x; ra[h * 4 + 1] = v.y; ra[h * 4 + 2] = v.z; ra[h * 4 + 3] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        ra[h * 4 + j] = (gm < M && gk + j < K) ? A[(size_t)gm * lda + gk + j] : 0.0f;
    }
  }
}

template <bool kAligned>
__device__ __forceinline__ void load_b(const float* __restrict__ B, int ldb,
                                       int K, int N, int k0, int n0,
                                       float (&rb)[8]) {
  // 16 k x 128 cols: thread t loads k = t>>5 and (t>>5)+8, cols (t&31)*4..
  const int r = threadIdx.x >> 5, c = (threadIdx.x & 31) * 4;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int gk = k0 + r + h * 8, gn = n0 + c;
    if (kAligned && gk < K && gn + 3 < N) {
      float4 v = __ldg(reinterpret_cast<const float4*>(B + (size_t)gk * ldb + gn));
      rb[h * 4 + 0] = v.x; rb[h * 4 + 1] = v.y; rb[h * 4 + 2] = v.z; rb[h * 4 + 3] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        rb[h * 4 + j] = (gk < K && gn + j < N) ? B[(size_t)gk * ldb + gn + j] : 0.0f;
    }
  }
}

template <bool kAligned>
__global__ void __launch_bounds__(NT, 2)
    sgemm_simt_kernel(const float* __restrict__ A, const float* __restrict__ B,
                      float* __restrict__ C, int M, int N, int K, int lda,
                      int ldb, int ldc) {
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;

  // accumulators as packed pairs (columns 2p, 2p+1 of row i): the inner
  // product is issued as FFMA2 (two FMAs per lane per instruction), which
  // halves the issue slots the FMAs take next to the shared-memory loads
  uint64_t acc2[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      acc2[i][j] = 0ull;

  float ra[8], rb[8];
  const int ar = threadIdx.x >> 2, ac = (threadIdx.x & 3) * 4;
  const int br = threadIdx.x >> 5, bc = (threadIdx.x & 31) * 4;
  auto stash = [&](int buf) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        As[buf][ac + j][ar + h * 64] = ra[h * 4 + j];
#pragma unroll
    for (int h = 0; h < 2; ++h)
      *reinterpret_cast<float4*>(&Bs[buf][br + h * 8][bc]) =
          make_float4(rb[h * 4], rb[h * 4 + 1], rb[h * 4 + 2], rb[h * 4 + 3]);
  };

  load_a<kAligned>(A, lda, M, K, m0, 0, ra);
  load_b<kAligned>(B, ldb, K, N, 0, n0, rb);
  stash(0);
  __syncthreads();

  const int nk = (K + BK - 1) / BK;
  for (int kt = 0; kt < nk; ++kt) {
    const int cur = kt & 1;
    if (kt + 1 < nk) {
      load_a<kAligned>(A, lda, M, K, m0, (kt + 1) * BK, ra);
      load_b<kAligned>(B, ldb, K, N, (kt + 1) * BK, n0, rb);
    }
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[cur][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[cur][k][ty * 4 + 64]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[cur][k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[cur][k][tx * 4 + 64]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      uint64_t b2[4];
      asm("mov.b64 %0, {%1, %2};" : "=l"(b2[0]) : "f"(b0.x), "f"(b0.y));
      asm("mov.b64 %0, {%1, %2};" : "=l"(b2[1]) : "f"(b0.z), "f"(b0.w));
      asm("mov.b64 %0, {%1, %2};" : "=l"(b2[2]) : "f"(b1.x), "f"(b1.y));
      asm("mov.b64 %0, {%1, %2};" : "=l"(b2[3]) : "f"(b1.z), "f"(b1.w));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint64_t a2;
        asm("mov.b64 %0, {%1, %1};" : "=l"(a2) : "f"(a[i]));
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[i][j]) : "l"(a2), "l"(b2[j]));
      }
    }
    if (kt + 1 < nk) {
      stash(cur ^ 1);
      __syncthreads();
    }
  }

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[i][2 * j]), "=f"(acc[i][2 * j + 1]) : "l"(acc2[i][j]));
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int gm = m0 + ty * 4 + (i & 3) + (i >> 2) * 64;
    if (gm >= M)
      continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int gn = n0 + tx * 4 + h * 64;
      float* dst = C + (size_t)gm * ldc + gn;
      if (kAligned && gn + 3 < N) {
        *reinterpret_cast<float4*>(dst) = make_float4(
            acc[i][h * 4], acc[i][h * 4 + 1], acc[i][h * 4 + 2], acc[i][h * 4 + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (gn + j < N)
            dst[j] = acc[i][h * 4 + j];
      }
    }
  }
}

}  // namespace

int sgemm_simt_launch(const float* A, const float* B, float* C, int M, int N,
                      int K, int lda, int ldb, int ldc, void* stream) {
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  bool aligned = ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0) &&
                 ((uintptr_t)C % 16 == 0) && lda % 4 == 0 && ldb % 4 == 0 &&
                 ldc % 4 == 0;
  if (aligned)
    sgemm_simt_kernel<true><<<grid, NT, 0, (cudaStream_t)stream>>>(
        A, B, C, M, N, K, lda, ldb, ldc);
  else
    sgemm_simt_kernel<false><<<grid, NT, 0, (cudaStream_t)stream>>>(
        A, B, C, M, N, K, lda, ldb, ldc);
  return (int)cudaGetLastError();
}

}  // namespace cafxg
