// FP-pipe peak probe: the denominator of the Mandelbrot roofline measured on
// the box instead of assumed. Each kernel runs 8 independent dependency chains
// per thread over a full-occupancy grid; prints lane-ops/s per instruction
// kind (a packed f32x2 instruction counts 2 lane-ops) and the SM clock seen.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_peak fp_peak.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CHAINS 8

template <int KIND>
__global__ void __launch_bounds__(256) probe(float* out, int iters, float a, float b) {
  float x[CHAINS * 2];
  double dx[CHAINS];
  uint32_t cnt[CHAINS] = {};
#pragma unroll
  for (int c = 0; c < CHAINS * 2; ++c)
    x[c] = threadIdx.x * 1e-3f + c;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c)
    dx[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if constexpr (KIND == 0) {  // scalar FADD x2 (two chains)
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[2 * c]) : "f"(a));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[2 * c + 1]) : "f"(a));
      } else if constexpr (KIND == 1) {  // scalar FMUL
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(x[2 * c]) : "f"(a));
        asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(x[2 * c + 1]) : "f"(a));
      } else if constexpr (KIND == 2) {  // packed FADD2
        asm volatile("{.reg .b64 r, s; mov.b64 r, {%0,%1}; mov.b64 s, {%2,%2};"
                     "add.rn.f32x2 r, r, s; mov.b64 {%0,%1}, r;}"
                     : "+f"(x[2 * c]), "+f"(x[2 * c + 1]) : "f"(a));
      } else if constexpr (KIND == 3) {  // packed FFMA2 (3 register operands)
        asm volatile("{.reg .b64 r, s, t; mov.b64 r, {%0,%1}; mov.b64 s, {%2,%2};"
                     "mov.b64 t, {%3,%3}; fma.rn.f32x2 r, r, s, t; mov.b64 {%0,%1}, r;}"
                     : "+f"(x[2 * c]), "+f"(x[2 * c + 1]) : "f"(a), "f"(b));
      } else if constexpr (KIND == 4) {  // scalar DADD
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(dx[c]) : "d"((double)a));
      } else if constexpr (KIND == 5) {  // scalar DMUL
        asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(dx[c]) : "d"((double)a));
      } else if constexpr (KIND >= 6) {
        // the Mandelbrot escape step's FP2 mix (7 packed ops, 2 pixels) on 4
        // independent pixel pairs per thread; KIND 7 adds the per-step
        // escape bookkeeping (2 x FSETP.OR + 2 x predicated IADD)
        if (c < (KIND == 8 ? 1 : KIND == 9 ? 2 : CHAINS / 2)) {
          float* z = &x[4 * c];
          if constexpr (KIND == 6)
            asm volatile(
                "{.reg .b64 X, Y, T, V, two, zz, C;"
                "mov.b64 X, {%0,%1}; mov.b64 Y, {%2,%3}; mov.b64 C, {%4,%4};"
                "mov.b64 zz, {%5,%5}; mov.b64 two, {%6,%6};"
                "fma.rn.f32x2 T, X, X, zz; fma.rn.f32x2 V, Y, Y, zz;"
                "sub.rn.f32x2 T, T, V; add.rn.f32x2 T, T, C; mul.rn.f32x2 V, X, Y;"
                "fma.rn.f32x2 Y, V, two, C; add.rn.f32x2 X, T, zz;"
                "mov.b64 {%0,%1}, X; mov.b64 {%2,%3}, Y;}"
                : "+f"(z[0]), "+f"(z[1]), "+f"(z[2]), "+f"(z[3])
                : "f"(a), "f"(0.0f), "f"(b));
          else
            asm volatile(
                "{.reg .b64 X, Y, T, V, two, zz, C; .reg .f32 s0, s1; .reg .pred q0, q1;"
                "setp.ne.u32 q0, %4, 0; setp.ne.u32 q1, %4, 7;"
                "mov.b64 X, {%0,%1}; mov.b64 Y, {%2,%3}; mov.b64 C, {%5,%5};"
                "mov.b64 zz, {%6,%6}; mov.b64 two, {%7,%7};"
                "fma.rn.f32x2 T, X, X, zz; fma.rn.f32x2 V, Y, Y, zz;"
                "sub.rn.f32x2 T, T, V; add.rn.f32x2 T, T, C; mul.rn.f32x2 V, X, Y;"
                "fma.rn.f32x2 Y, V, two, C; add.rn.f32x2 X, T, zz;"
                "mov.b64 {s0, s1}, X;"
                "setp.gt.or.f32 q0, s0, 0f40800000, q0; setp.gt.or.f32 q1, s1, 0f40800000, q1;"
                "@!q0 add.u32 %4, %4, 1; @!q1 add.u32 %4, %4, 3;"
                "mov.b64 {%0,%1}, X; mov.b64 {%2,%3}, Y;}"
                : "+f"(z[0]), "+f"(z[1]), "+f"(z[2]), "+f"(z[3]), "+r"(cnt[c])
                : "f"(a), "f"(0.0f), "f"(b));
        }
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS * 2; ++c)
    s += x[c];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c)
    s += (float)dx[c] + (float)cnt[c];
  if (s == 12345.678f)
    out[0] = s;
}

template <int KIND>
double run(const char* name, double lane_ops_per_iter_thread, int sms) {
  float* out;
  cudaMalloc(&out, 4);
  int blocks = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, probe<KIND>, 256, 0);
  int grid = sms * blocks;
  int iters = 20000;
  probe<KIND><<<grid, 256>>>(out, 100, 1.0000001f, 0.5f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<KIND><<<grid, 256>>>(out, iters, 1.0000001f, 0.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)grid * 256 * iters * lane_ops_per_iter_thread;
  double rate = ops / (ms * 1e-3) / 1e12;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"kind\": \"%s\", \"lane_Tops\": %.3f, \"per_sm_per_clk_at_max\": %.1f, "
         "\"ms\": %.3f, \"grid\": %d}\n",
         name, rate, rate * 1e12 / sms / (clk * 1e3), ms, grid);
  cudaFree(out);
  return rate;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("FADD scalar", 2.0 * CHAINS, sms);
  run<1>("FMUL scalar", 2.0 * CHAINS, sms);
  run<2>("FADD2 packed", 2.0 * CHAINS, sms);
  run<3>("FFMA2 packed (2 flop/lane-op)", 2.0 * CHAINS, sms);
  run<4>("DADD", 1.0 * CHAINS, sms);
  run<5>("DMUL", 1.0 * CHAINS, sms);
  // 4 chains x 7 FP2 x 2 lanes per iteration
  run<6>("escape-step FP2 mix (lane-ops of 7 FP2)", 4.0 * 7 * 2, sms);
  run<7>("escape-step FP2 mix + FSETP/IADD bookkeeping", 4.0 * 7 * 2, sms);
  run<8>("escape-step + bookkeeping, 1 chain per thread", 1.0 * 7 * 2, sms);
  run<9>("escape-step + bookkeeping, 2 chains per thread", 2.0 * 7 * 2, sms);
  return 0;
}
