// Escape-time (Mandelbrot) kernels for sm_100a.
//
// Reference semantics: cafx::bench::mandelbrot_cell
// (/root/reference/proj/src/bench/bench.cpp:367-379), generalised per
// SURVEY.md §8a row a2 (include/cafxg.h documents the coordinate contract).
//
// Design:
//  * persistent grid; each warp pulls 512-pixel chunks (never straddling a
//    row) from a global cursor and every lane carries several independent
//    pixels ("slots"). In fp32 two slots share the halves of 64-bit registers
//    and each escape step is issued as packed FADD2/FMUL2/FFMA2 instructions
//    (f32x2, new in sm_100): 7 packed FP instructions advance 2 pixels by one
//    iteration; a lane runs two such pairs (4 pixels) so each warp has two
//    independent dependency chains in flight;
//  * bit-exact counting without per-step branches: a sticky escape predicate
//    (FSETP.OR) and a counter that stops at the first escape. After the first
//    escape z keeps iterating (to inf/NaN) but the predicate never clears, so
//    `count = escaped ? steps_before + 1 : steps` equals the reference's
//    early-exit loop, capped at max_iter (an escape exactly at max_iter also
//    returns max_iter, as bench.cpp:378);
//  * refill: every `ksteps` iterations the warp votes; lanes whose pixel is
//    finished store the count and take the next pixel from the warp's chunk,
//    so no lane idles behind a slow neighbour (divergence-free main loop);
//  * every FP op is an explicit round-to-nearest `.rn` PTX op, so nothing can
//    contract the reference's separate mul and add into one FMA.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "mandelbrot.cuh"

namespace cafxg {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// ---- the escape-iteration block ----------------------------------------------
// kSteps iterations of the reference loop (bench.cpp:370-377) for a lane's
// slots, written as one PTX block so the escape bookkeeping stays in
// predicates: per slot and step one `setp.gt.or` (sticky escape flag) and one
// predicated add (the count stops at the first escape). Reference order, with
// the squares shared between the escape test and the next step exactly as the
// compiled reference does:
//   nr = (zr*zr - zi*zi) + re ; ni = (2*zr)*zi + im ; escape if nr^2+ni^2 > 4
//
// Two ptxas facts shape the text:
//  * ptxas 12.9 contracts `mul.rn.f32x2` + `add.rn.f32x2` into FFMA2 in spite
//    of the explicit rounding (checked in SASS; scalar .rn is respected).
//    Squares are therefore formed as fma(a, a, z) with z a RUNTIME +0.0
//    (MLaunch::zero): fl(a*a + 0) == fl(a*a) and an FFMA2 result is never
//    fused further;
//  * the fast step folds `(2*zr)*zi + im` into fma(zr*zi, 2, im): fl(2zr)*zi
//    rounds to 2*fl(zr*zi) (power-of-two scaling commutes with rounding) and
//    fl(2v + im) with 2v exact is one fma. Bit-identical unless fl(zr*zi) is
//    subnormal, which the host rules out per request; the
//    `exact` step keeps the reference's 8 separate operations.

// One fp32 pair step. Register names: X zr, Y zi, Q zr^2, W zi^2 (packed
// state), C cr, D ci (packed inputs), T/V/S temporaries, A0/A1 unpacked sums,
// P0/P1 sticky predicates, N0/N1 counts.
#define CAFXG_F32_FAST(X, Y, Q, W, C, D, T, V, S, A0, A1, P0, P1, N0, N1) \
  "sub.rn.f32x2 " T ", " Q ", " W ";\n\t"                                 \
  "add.rn.f32x2 " T ", " T ", " C ";\n\t"                                 \
  "mul.rn.f32x2 " V ", " X ", " Y ";\n\t"                                 \
  "fma.rn.f32x2 " Y ", " V ", two, " D ";\n\t"                            \
  "mov.b64 " X ", " T ";\n\t"                                             \
  "fma.rn.f32x2 " Q ", " X ", " X ", zz;\n\t"                             \
  "fma.rn.f32x2 " W ", " Y ", " Y ", zz;\n\t"                             \
  "add.rn.f32x2 " S ", " Q ", " W ";\n\t"                                 \
  "mov.b64 {" A0 ", " A1 "}, " S ";\n\t"                                  \
  "setp.gt.or.f32 " P0 ", " A0 ", 0f40800000, " P0 ";\n\t"                \
  "setp.gt.or.f32 " P1 ", " A1 ", 0f40800000, " P1 ";\n\t"                \
  "@!" P0 " add.u32 " N0 ", " N0 ", 1;\n\t"                               \
  "@!" P1 " add.u32 " N1 ", " N1 ", 1;\n\t"

#define CAFXG_F32_EXACT(X, Y, Q, W, C, D, T, V, S, A0, A1, P0, P1, N0, N1) \
  "sub.rn.f32x2 " T ", " Q ", " W ";\n\t"                                  \
  "add.rn.f32x2 " T ", " T ", " C ";\n\t"                                  \
  "add.rn.f32x2 " V ", " X ", " X ";\n\t"                                  \
  "fma.rn.f32x2 " V ", " V ", " Y ", zz;\n\t"                              \
  "add.rn.f32x2 " Y ", " V ", " D ";\n\t"                                  \
  "mov.b64 " X ", " T ";\n\t"                                              \
  "fma.rn.f32x2 " Q ", " X ", " X ", zz;\n\t"                              \
  "fma.rn.f32x2 " W ", " Y ", " Y ", zz;\n\t"                              \
  "add.rn.f32x2 " S ", " Q ", " W ";\n\t"                                  \
  "mov.b64 {" A0 ", " A1 "}, " S ";\n\t"                                   \
  "setp.gt.or.f32 " P0 ", " A0 ", 0f40800000, " P0 ";\n\t"                 \
  "setp.gt.or.f32 " P1 ", " A1 ", 0f40800000, " P1 ";\n\t"                 \
  "@!" P0 " add.u32 " N0 ", " N0 ", 1;\n\t"                                \
  "@!" P1 " add.u32 " N1 ", " N1 ", 1;\n\t"

// Both pairs of a lane, interleaved (two independent chains).
// operands: %0..%3 pair A {zr, zi, zr^2, zi^2}; %4..%7 pair B; %8..%11
// counts (A0, A1, B0, B1; bit 31 = sticky escape flag, max_iter <= 2^30
// keeps it free); %12 crA, %13 ciA, %14 crB, %15 ciB; %16 runtime zero;
// %17 2.0f.
#define CAFXG_F32_STEP2(STEP)                                                  \
  STEP("%0", "%1", "%2", "%3", "%12", "%13", "tA", "vA", "sA", "a0", "a1", "pA0", \
       "pA1", "%8", "%9")                                                       \
  STEP("%4", "%5", "%6", "%7", "%14", "%15", "tB", "vB", "sB", "b0", "b1", "pB0", \
       "pB1", "%10", "%11")

#define CAFXG_F32_PROLOGUE                                                 \
  "{\n\t.reg .b64 tA, vA, sA, tB, vB, sB, two, zz;\n\t"                    \
  ".reg .f32 a0, a1, b0, b1;\n\t.reg .pred pA0, pA1, pB0, pB1;\n\t"        \
  "mov.b64 zz, {%16, %16};\n\tmov.b64 two, {%17, %17};\n\t"                \
  "setp.lt.s32 pA0, %8, 0;\n\tsetp.lt.s32 pA1, %9, 0;\n\t"                 \
  "setp.lt.s32 pB0, %10, 0;\n\tsetp.lt.s32 pB1, %11, 0;\n\t"

#define CAFXG_F32_EPILOGUE                                                 \
  "@pA0 or.b32 %8, %8, 0x80000000;\n\t@pA1 or.b32 %9, %9, 0x80000000;\n\t" \
  "@pB0 or.b32 %10, %10, 0x80000000;\n\t@pB1 or.b32 %11, %11, 0x80000000;\n\t}"

#define CAFXG_X4(S) S S S S
#define CAFXG_X8(S) CAFXG_X4(S) CAFXG_X4(S)
#define CAFXG_X16(S) CAFXG_X4(S) CAFXG_X4(S) CAFXG_X4(S) CAFXG_X4(S)
#define CAFXG_X12(S) CAFXG_X8(S) CAFXG_X4(S)
#define CAFXG_X20(S) CAFXG_X16(S) CAFXG_X4(S)
#define CAFXG_X24(S) CAFXG_X16(S) CAFXG_X8(S)
#define CAFXG_X28(S) CAFXG_X24(S) CAFXG_X4(S)
#define CAFXG_X32(S) CAFXG_X16(S) CAFXG_X16(S)
#define CAFXG_X40(S) CAFXG_X32(S) CAFXG_X8(S)
#define CAFXG_X48(S) CAFXG_X32(S) CAFXG_X16(S)
#define CAFXG_X56(S) CAFXG_X48(S) CAFXG_X8(S)
#define CAFXG_X64(S) CAFXG_X32(S) CAFXG_X32(S)

// Expands BODY(CAFXG_Xk) for the compile-time step count K (one unrolled
// PTX block of K steps).
#define CAFXG_STEPS_SWITCH(K, BODY)                    \
  if constexpr (K == 4) { BODY(CAFXG_X4); }            \
  else if constexpr (K == 8) { BODY(CAFXG_X8); }       \
  else if constexpr (K == 12) { BODY(CAFXG_X12); }     \
  else if constexpr (K == 16) { BODY(CAFXG_X16); }     \
  else if constexpr (K == 20) { BODY(CAFXG_X20); }     \
  else if constexpr (K == 24) { BODY(CAFXG_X24); }     \
  else if constexpr (K == 28) { BODY(CAFXG_X28); }     \
  else if constexpr (K == 32) { BODY(CAFXG_X32); }     \
  else if constexpr (K == 40) { BODY(CAFXG_X40); }     \
  else if constexpr (K == 48) { BODY(CAFXG_X48); }     \
  else if constexpr (K == 56) { BODY(CAFXG_X56); }     \
  else { static_assert(K == 64, "unsupported step count"); BODY(CAFXG_X64); }

#define CAFXG_F32_OPERANDS                                                     \
  : "+l"(zr[0]), "+l"(zi[0]), "+l"(zr2[0]), "+l"(zi2[0]), "+l"(zr[1]),         \
    "+l"(zi[1]), "+l"(zr2[1]), "+l"(zi2[1]), "+r"(n[0]), "+r"(n[1]),           \
    "+r"(n[2]), "+r"(n[3])                                                     \
  : "l"(cr[0]), "l"(ci[0]), "l"(cr[1]), "l"(ci[1]), "f"(zero), "f"(2.0f)

// ---- unchecked blocks (deferred escape test) --------------------------------
// The same steps without the per-step test: 6 packed FP ops per pair and
// step (7 with the reference's 8-op form). Escape is tested once per block;
// see mandel_deferred_kernel for why that is exact.
#define CAFXG_F32_FREE_FAST(X, Y, Q, W, C, D, T, V) \
  "sub.rn.f32x2 " T ", " Q ", " W ";\n\t"           \
  "add.rn.f32x2 " T ", " T ", " C ";\n\t"           \
  "mul.rn.f32x2 " V ", " X ", " Y ";\n\t"           \
  "fma.rn.f32x2 " Y ", " V ", two, " D ";\n\t"      \
  "mov.b64 " X ", " T ";\n\t"                       \
  "fma.rn.f32x2 " Q ", " X ", " X ", zz;\n\t"       \
  "fma.rn.f32x2 " W ", " Y ", " Y ", zz;\n\t"

#define CAFXG_F32_FREE_EXACT(X, Y, Q, W, C, D, T, V) \
  "sub.rn.f32x2 " T ", " Q ", " W ";\n\t"            \
  "add.rn.f32x2 " T ", " T ", " C ";\n\t"            \
  "add.rn.f32x2 " V ", " X ", " X ";\n\t"            \
  "fma.rn.f32x2 " V ", " V ", " Y ", zz;\n\t"        \
  "add.rn.f32x2 " Y ", " V ", " D ";\n\t"            \
  "mov.b64 " X ", " T ";\n\t"                        \
  "fma.rn.f32x2 " Q ", " X ", " X ", zz;\n\t"        \
  "fma.rn.f32x2 " W ", " Y ", " Y ", zz;\n\t"

#define CAFXG_F32_FREE2(STEP)                                       \
  STEP("%0", "%1", "%2", "%3", "%8", "%9", "tA", "vA")              \
  STEP("%4", "%5", "%6", "%7", "%10", "%11", "tB", "vB")

#define CAFXG_F32_FREE_PROLOGUE                                     \
  "{\n\t.reg .b64 tA, vA, tB, vB, two, zz;\n\t"                     \
  "mov.b64 zz, {%12, %12};\n\tmov.b64 two, {%13, %13};\n\t"
#define CAFXG_F32_FREE_EPILOGUE "}"
#define CAFXG_F32_FREE_OPERANDS                                             \
  : "+l"(zr[0]), "+l"(zi[0]), "+l"(zr2[0]), "+l"(zi2[0]), "+l"(zr[1]),      \
    "+l"(zi[1]), "+l"(zr2[1]), "+l"(zi2[1])                                 \
  : "l"(cr[0]), "l"(ci[0]), "l"(cr[1]), "l"(ci[1]), "f"(zero), "f"(2.0f)

__device__ __forceinline__ uint64_t set_half(uint64_t v, int hi, float f) {
  uint64_t b = __float_as_uint(f);
  return hi ? ((v & 0xffffffffull) | (b << 32)) : ((v & 0xffffffff00000000ull) | b);
}
__device__ __forceinline__ float get_half(uint64_t v, int hi) {
  return __uint_as_float(hi ? (uint32_t)(v >> 32) : (uint32_t)v);
}

struct F32Slots {
  static constexpr int kSlots = 4;  // two packed pairs per lane
  using C = float;                  // coordinate table element
  uint64_t zr[2] = {}, zi[2] = {}, zr2[2] = {}, zi2[2] = {}, cr[2] = {}, ci[2] = {};
  float zero;

  template <int kSteps, bool kExact>
  __device__ __forceinline__ void run(uint32_t (&n)[kSlots]) {
#define CAFXG_B_FAST(X) asm volatile(CAFXG_F32_PROLOGUE X(CAFXG_F32_STEP2(CAFXG_F32_FAST)) \
                                         CAFXG_F32_EPILOGUE CAFXG_F32_OPERANDS)
#define CAFXG_B_EXACT(X) asm volatile(CAFXG_F32_PROLOGUE X(CAFXG_F32_STEP2(CAFXG_F32_EXACT)) \
                                          CAFXG_F32_EPILOGUE CAFXG_F32_OPERANDS)
    if constexpr (kExact) {
      CAFXG_STEPS_SWITCH(kSteps, CAFXG_B_EXACT)
    } else {
      CAFXG_STEPS_SWITCH(kSteps, CAFXG_B_FAST)
    }
#undef CAFXG_B_FAST
#undef CAFXG_B_EXACT
  }
  template <int kSteps, bool kExact>
  __device__ __forceinline__ void run_free() {
#define CAFXG_B_FAST(X) asm volatile(CAFXG_F32_FREE_PROLOGUE X(CAFXG_F32_FREE2(CAFXG_F32_FREE_FAST)) \
                                         CAFXG_F32_FREE_EPILOGUE CAFXG_F32_FREE_OPERANDS)
#define CAFXG_B_EXACT(X) asm volatile(CAFXG_F32_FREE_PROLOGUE X(CAFXG_F32_FREE2(CAFXG_F32_FREE_EXACT)) \
                                          CAFXG_F32_FREE_EPILOGUE CAFXG_F32_FREE_OPERANDS)
    if constexpr (kExact) {
      CAFXG_STEPS_SWITCH(kSteps, CAFXG_B_EXACT)
    } else {
      CAFXG_STEPS_SWITCH(kSteps, CAFXG_B_FAST)
    }
#undef CAFXG_B_FAST
#undef CAFXG_B_EXACT
  }
  // slot s lives in half (s & 1) of pair (s >> 1)
  __device__ __forceinline__ void start(int s, float fr, float fi) {
    const int p = s >> 1, h = s & 1;
    cr[p] = set_half(cr[p], h, fr);
    ci[p] = set_half(ci[p], h, fi);
    zr[p] = set_half(zr[p], h, 0.0f);
    zi[p] = set_half(zi[p], h, 0.0f);
    zr2[p] = set_half(zr2[p], h, 0.0f);
    zi2[p] = set_half(zi2[p], h, 0.0f);
  }
  // resumes slot s at a saved z; the squares are recomputed exactly as the
  // step forms them (fma(a, a, +0) == fl(a * a))
  __device__ __forceinline__ void resume(int s, float r, float i, float fr, float fi) {
    const int p = s >> 1, h = s & 1;
    cr[p] = set_half(cr[p], h, fr);
    ci[p] = set_half(ci[p], h, fi);
    zr[p] = set_half(zr[p], h, r);
    zi[p] = set_half(zi[p], h, i);
    zr2[p] = set_half(zr2[p], h, __fmul_rn(r, r));
    zi2[p] = set_half(zi2[p], h, __fmul_rn(i, i));
  }
  __device__ __forceinline__ float zr_of(int s) const { return get_half(zr[s >> 1], s & 1); }
  __device__ __forceinline__ float zi_of(int s) const { return get_half(zi[s >> 1], s & 1); }
  __device__ __forceinline__ float cr_of(int s) const { return get_half(cr[s >> 1], s & 1); }
  __device__ __forceinline__ float ci_of(int s) const { return get_half(ci[s >> 1], s & 1); }
  // mid-block checkpoint (deferred kernel): both pairs' packed z per lane
  struct Mid {
    uint64_t zr[2][32], zi[2][32];
  };
  __device__ __forceinline__ void save_mid(Mid& m, uint32_t lane) const {
    m.zr[0][lane] = zr[0];
    m.zr[1][lane] = zr[1];
    m.zi[0][lane] = zi[0];
    m.zi[1][lane] = zi[1];
  }
  static __device__ __forceinline__ float mid_zr(const Mid& m, int s, uint32_t lane) {
    return get_half(m.zr[s >> 1][lane], s & 1);
  }
  static __device__ __forceinline__ float mid_zi(const Mid& m, int s, uint32_t lane) {
    return get_half(m.zi[s >> 1][lane], s & 1);
  }
  // the block-end test on a saved z: fl(fl(zr^2) + fl(zi^2)) > 4 or NaN
  static __device__ __forceinline__ bool escaped_at(float r, float i) {
    return !(__fadd_rn(__fmul_rn(r, r), __fmul_rn(i, i)) <= 4.0f);
  }
  // bit s: fl(zr^2 + zi^2) > 4 or NaN (an orbit that overflowed)
  __device__ __forceinline__ uint32_t escaped() const {
    uint32_t m = 0;
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
      float S = __fadd_rn(get_half(zr2[s >> 1], s & 1), get_half(zi2[s >> 1], s & 1));
      m |= (!(S <= 4.0f)) ? (1u << s) : 0u;
    }
    return m;
  }
};

// fp64: two scalar slots; scalar `.rn` ops are never contracted by ptxas.
#define CAFXG_F64_STEP_FAST(X, Y, Q, W, C, D, P, N)                 \
  "sub.rn.f64 t, " Q ", " W ";\n\t"                                  \
  "add.rn.f64 t, t, " C ";\n\t"                                      \
  "mul.rn.f64 v, " X ", " Y ";\n\t"                                  \
  "fma.rn.f64 " Y ", v, 0d4000000000000000, " D ";\n\t"              \
  "mov.f64 " X ", t;\n\t"                                            \
  "mul.rn.f64 " Q ", " X ", " X ";\n\t"                              \
  "mul.rn.f64 " W ", " Y ", " Y ";\n\t"                              \
  "add.rn.f64 s, " Q ", " W ";\n\t"                                  \
  "setp.gt.or.f64 " P ", s, 0d4010000000000000, " P ";\n\t"          \
  "@!" P " add.u32 " N ", " N ", 1;\n\t"

#define CAFXG_F64_STEP_EXACT(X, Y, Q, W, C, D, P, N)                \
  "sub.rn.f64 t, " Q ", " W ";\n\t"                                  \
  "add.rn.f64 t, t, " C ";\n\t"                                      \
  "add.rn.f64 v, " X ", " X ";\n\t"                                  \
  "mul.rn.f64 v, v, " Y ";\n\t"                                      \
  "add.rn.f64 " Y ", v, " D ";\n\t"                                  \
  "mov.f64 " X ", t;\n\t"                                            \
  "mul.rn.f64 " Q ", " X ", " X ";\n\t"                              \
  "mul.rn.f64 " W ", " Y ", " Y ";\n\t"                              \
  "add.rn.f64 s, " Q ", " W ";\n\t"                                  \
  "setp.gt.or.f64 " P ", s, 0d4010000000000000, " P ";\n\t"          \
  "@!" P " add.u32 " N ", " N ", 1;\n\t"

#define CAFXG_F64_PAIR(STEP)                                             \
  STEP("%0", "%1", "%2", "%3", "%10", "%11", "p0", "%8")                 \
  STEP("%4", "%5", "%6", "%7", "%12", "%13", "p1", "%9")

#define CAFXG_F64_PROLOGUE                                               \
  "{\n\t.reg .f64 t, v, s;\n\t.reg .pred p0, p1;\n\t"                    \
  "setp.lt.s32 p0, %8, 0;\n\tsetp.lt.s32 p1, %9, 0;\n\t"
#define CAFXG_F64_EPILOGUE                                               \
  "@p0 or.b32 %8, %8, 0x80000000;\n\t"                                 \
  "@p1 or.b32 %9, %9, 0x80000000;\n\t}"
#define CAFXG_F64_OPERANDS                                               \
  : "+d"(zr.x), "+d"(zi.x), "+d"(zr2.x), "+d"(zi2.x), "+d"(zr.y),         \
    "+d"(zi.y), "+d"(zr2.y), "+d"(zi2.y), "+r"(n[0]), "+r"(n[1])          \
  : "d"(cr.x), "d"(ci.x), "d"(cr.y), "d"(ci.y)

#define CAFXG_F64_FREE_FAST(X, Y, Q, W, C, D)           \
  "sub.rn.f64 t, " Q ", " W ";\n\t"                      \
  "add.rn.f64 t, t, " C ";\n\t"                          \
  "mul.rn.f64 v, " X ", " Y ";\n\t"                      \
  "fma.rn.f64 " Y ", v, 0d4000000000000000, " D ";\n\t"  \
  "mov.f64 " X ", t;\n\t"                                \
  "mul.rn.f64 " Q ", " X ", " X ";\n\t"                  \
  "mul.rn.f64 " W ", " Y ", " Y ";\n\t"

#define CAFXG_F64_FREE_EXACT(X, Y, Q, W, C, D)          \
  "sub.rn.f64 t, " Q ", " W ";\n\t"                      \
  "add.rn.f64 t, t, " C ";\n\t"                          \
  "add.rn.f64 v, " X ", " X ";\n\t"                      \
  "mul.rn.f64 v, v, " Y ";\n\t"                          \
  "add.rn.f64 " Y ", v, " D ";\n\t"                      \
  "mov.f64 " X ", t;\n\t"                                \
  "mul.rn.f64 " Q ", " X ", " X ";\n\t"                  \
  "mul.rn.f64 " W ", " Y ", " Y ";\n\t"

#define CAFXG_F64_FREE2(STEP)                          \
  STEP("%0", "%1", "%2", "%3", "%8", "%9")             \
  STEP("%4", "%5", "%6", "%7", "%10", "%11")
#define CAFXG_F64_FREE_PROLOGUE "{\n\t.reg .f64 t, v;\n\t"
#define CAFXG_F64_FREE_OPERANDS                                          \
  : "+d"(zr.x), "+d"(zi.x), "+d"(zr2.x), "+d"(zi2.x), "+d"(zr.y),         \
    "+d"(zi.y), "+d"(zr2.y), "+d"(zi2.y)                                  \
  : "d"(cr.x), "d"(ci.x), "d"(cr.y), "d"(ci.y)

struct F64Slots {
  static constexpr int kSlots = 2;
  using C = double;
  double2 zr{}, zi{}, zr2{}, zi2{}, cr{}, ci{};
  float zero;

  template <int kSteps, bool kExact>
  __device__ __forceinline__ void run(uint32_t (&n)[kSlots]) {
#define CAFXG_B_FAST(X) asm volatile(CAFXG_F64_PROLOGUE X(CAFXG_F64_PAIR(CAFXG_F64_STEP_FAST)) \
                                         CAFXG_F64_EPILOGUE CAFXG_F64_OPERANDS)
#define CAFXG_B_EXACT(X) asm volatile(CAFXG_F64_PROLOGUE X(CAFXG_F64_PAIR(CAFXG_F64_STEP_EXACT)) \
                                          CAFXG_F64_EPILOGUE CAFXG_F64_OPERANDS)
    if constexpr (kExact) {
      CAFXG_STEPS_SWITCH(kSteps, CAFXG_B_EXACT)
    } else {
      CAFXG_STEPS_SWITCH(kSteps, CAFXG_B_FAST)
    }
#undef CAFXG_B_FAST
#undef CAFXG_B_EXACT
  }
  template <int kSteps, bool kExact>
  __device__ __forceinline__ void run_free() {
#define CAFXG_B_FAST(X) asm volatile(CAFXG_F64_FREE_PROLOGUE X(CAFXG_F64_FREE2(CAFXG_F64_FREE_FAST)) \
                                         "}" CAFXG_F64_FREE_OPERANDS)
#define CAFXG_B_EXACT(X) asm volatile(CAFXG_F64_FREE_PROLOGUE X(CAFXG_F64_FREE2(CAFXG_F64_FREE_EXACT)) \
                                          "}" CAFXG_F64_FREE_OPERANDS)
    if constexpr (kExact) {
      CAFXG_STEPS_SWITCH(kSteps, CAFXG_B_EXACT)
    } else {
      CAFXG_STEPS_SWITCH(kSteps, CAFXG_B_FAST)
    }
#undef CAFXG_B_FAST
#undef CAFXG_B_EXACT
  }
  __device__ __forceinline__ void start(int s, double xr, double xi) {
    if (s == 0) {
      cr.x = xr; ci.x = xi; zr.x = zi.x = zr2.x = zi2.x = 0.0;
    } else {
      cr.y = xr; ci.y = xi; zr.y = zi.y = zr2.y = zi2.y = 0.0;
    }
  }
  __device__ __forceinline__ void resume(int s, double r, double i, double xr, double xi) {
    if (s == 0) {
      cr.x = xr; ci.x = xi; zr.x = r; zi.x = i;
      zr2.x = __dmul_rn(r, r); zi2.x = __dmul_rn(i, i);
    } else {
      cr.y = xr; ci.y = xi; zr.y = r; zi.y = i;
      zr2.y = __dmul_rn(r, r); zi2.y = __dmul_rn(i, i);
    }
  }
  __device__ __forceinline__ double zr_of(int s) const { return s ? zr.y : zr.x; }
  __device__ __forceinline__ double zi_of(int s) const { return s ? zi.y : zi.x; }
  __device__ __forceinline__ double cr_of(int s) const { return s ? cr.y : cr.x; }
  __device__ __forceinline__ double ci_of(int s) const { return s ? ci.y : ci.x; }
  struct Mid {
    double2 zr[32], zi[32];
  };
  __device__ __forceinline__ void save_mid(Mid& m, uint32_t lane) const {
    m.zr[lane] = zr;
    m.zi[lane] = zi;
  }
  static __device__ __forceinline__ double mid_zr(const Mid& m, int s, uint32_t lane) {
    return s ? m.zr[lane].y : m.zr[lane].x;
  }
  static __device__ __forceinline__ double mid_zi(const Mid& m, int s, uint32_t lane) {
    return s ? m.zi[lane].y : m.zi[lane].x;
  }
  static __device__ __forceinline__ bool escaped_at(double r, double i) {
    return !(__dadd_rn(__dmul_rn(r, r), __dmul_rn(i, i)) <= 4.0);
  }
  __device__ __forceinline__ uint32_t escaped() const {
    double s0 = __dadd_rn(zr2.x, zi2.x), s1 = __dadd_rn(zr2.y, zi2.y);
    return ((!(s0 <= 4.0)) ? 1u : 0u) | ((!(s1 <= 4.0)) ? 2u : 0u);
  }
};

__device__ __forceinline__ const MTile* tile_ptr(const MLaunch& L, uint32_t t) {
  return L.n <= (uint32_t)kInlineTiles ? &L.inl[t] : &L.tiles[t];
}

__device__ __forceinline__ uint32_t find_tile(const MLaunch& L, uint32_t chunk) {
  uint32_t lo = 0, hi = L.n - 1;
  while (lo < hi) {
    uint32_t mid = (lo + hi + 1) >> 1;
    if (tile_ptr(L, mid)->chunk_begin <= chunk)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Coordinates as the oracle computes them (cafx_oracle.c oracle_coord):
// lo + ((i + s) * span) / n in fp64 with IEEE rounding, then rounded to the
// request precision. Computed once per column / row by the prologue kernel.
__device__ __forceinline__ double grid_coord(double lo, double span, double s,
                                             uint32_t i, uint32_t n) {
  double k = __dadd_rn((double)i, s);
  return __dadd_rn(lo, __ddiv_rn(__dmul_rn(k, span), (double)n));
}

template <class T>
__global__ void __launch_bounds__(256)
    coords_kernel(const __grid_constant__ MLaunch L) {
  const MTile* t = tile_ptr(L, blockIdx.y);
  T* cx = static_cast<T*>(t->cx);
  T* cy = static_cast<T*>(t->cy);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < t->ncols + t->nrows;
       i += gridDim.x * blockDim.x) {
    if (i < t->ncols)
      cx[i] = (T)grid_coord(t->x0, t->xspan, t->s, t->col0 + i, t->width);
    else
      cy[i - t->ncols] =
          (T)grid_coord(t->y0, t->yspan, t->s, t->row0 + (i - t->ncols), t->height);
  }
}

// ---- work distribution --------------------------------------------------------
// Warp-uniform cursor over columns [cur, cend) of one row of one tile. Chunks
// never straddle rows, so everything a new pixel needs besides its column
// coordinate is chunk state held in registers: the row's imaginary part, the
// column table and the output row base. refill() hands the next pixels to
// the lane slots that are free (bit s of `live` clear).
template <class Slots, int kMode>
struct Feeder {
  static constexpr bool kInlineCoords = kMode >= 1;
  using Cd = typename Slots::C;
  static constexpr int NS = Slots::kSlots;
  uint32_t cur = 0, cend = 0, orow = 0;
  uint32_t c0 = 0;            // first column of the chunk (inline mode)
  const Cd* cxp = nullptr;    // column table (table mode)
  Cd ci_row = Cd(0);
  bool exhausted = false;

  // Inline-coordinate launches: the warp's real parts of its current chunk,
  // computed by all 32 lanes when the chunk is claimed (4 per lane, the
  // fp64 divides at full SIMT width) instead of per refilled slot inside the
  // refill's divergent branches (cfg1: every refill round paid up to one
  // masked fp64 divide sequence per slot for a handful of pixels).
  __device__ __forceinline__ static Cd* chunk_table() {
    __shared__ Cd tab[kMandelThreads / 32][kChunkPx];
    return tab[threadIdx.x >> 5];
  }

  __device__ __forceinline__ void refill(const MLaunch& L, Slots& sl, uint32_t (&n)[NS],
                                         uint32_t (&o)[NS], uint32_t& live, uint32_t lt_mask) {
    const uint32_t lane = threadIdx.x & 31u;
    while (true) {
      uint32_t b[NS];
      uint32_t want = 0;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        b[s] = __ballot_sync(kFull, !(live >> s & 1u));
        want += __popc(b[s]);
      }
      if (want == 0 || exhausted)
        return;
      if (cur == cend) {
        uint32_t c = 0;
        if (lane == 0)
          c = atomicAdd(&L.sched[0], 1u);
        c = __shfl_sync(kFull, c, 0);
        if (c >= L.total_chunks) {
          exhausted = true;
          return;
        }
        const uint32_t ti = find_tile(L, c);
        const MTile* T = tile_ptr(L, ti);
        uint32_t local = c - T->chunk_begin;
        uint32_t cpr = T->chunks_per_row;
        uint32_t crow = local / cpr;
        uint32_t ncols = T->ncols;
        constexpr uint32_t kChunk = kChunkPx;
        cur = (local - crow * cpr) * kChunk;
        cend = min(cur + kChunk, ncols);
        if constexpr (kInlineCoords) {
          ci_row = (Cd)grid_coord(T->y0, T->yspan, T->s, T->row0 + crow, T->height);
          Cd* tab = chunk_table();
          __syncwarp();  // the previous chunk's entries are no longer read
#pragma unroll
          for (uint32_t j = lane; j < kChunkPx; j += 32)
            if (cur + j < cend)
              tab[j] = (Cd)grid_coord(T->x0, T->xspan, T->s, T->col0 + cur + j, T->width);
          __syncwarp();
          c0 = cur;
        } else {
          cxp = static_cast<const Cd*>(T->cx);
          ci_row = __ldg(static_cast<const Cd*>(T->cy) + crow);
        }
        orow = T->out_off + crow * ncols;
        if constexpr (kMode == 2)
          orow |= ti << kDirectShift;
        continue;
      }
      const uint32_t avail = cend - cur;
      uint32_t base = 0;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const uint32_t r = base + __popc(b[s] & lt_mask);
        if (!(live >> s & 1u) && r < avail) {
          Cd cr;
          if constexpr (kInlineCoords)
            cr = chunk_table()[cur - c0 + r];
          else
            cr = __ldg(cxp + cur + r);
          sl.start(s, cr, ci_row);
          n[s] = 0;
          o[s] = orow + cur + r;
          live |= 1u << s;
        }
        base += __popc(b[s]);
      }
      cur += min(want, avail);
      if (want <= avail)
        return;  // every free slot got a pixel (skips a round of ballots)
    }
  }
};

// ---- direct reply -------------------------------------------------------------
// Small batches (MLaunch::direct) skip the separate reply-scatter launch. Each
// warp counts the pixels it finishes per tile in shared memory (no fences on
// the per-round path); when the warp exits, it publishes its counts with one
// fence and one global atomic per tile it touched, and the warp whose count
// completes a tile copies the tile from the staging buffer (L2-resident, just
// written) to its pinned host reply, 8 x 16-byte loads in flight per lane.
// Ordering: stores -> __threadfence -> count (release); count ->
// __threadfence -> __ldcg of the tile (acquire).
__device__ __forceinline__ uint32_t* direct_counts() {
  __shared__ uint32_t cnt[kMandelThreads / 32][kInlineTiles];
  return cnt[threadIdx.x >> 5];
}

__device__ __forceinline__ void direct_begin() {
  direct_counts()[threadIdx.x & 31u] = 0;  // kInlineTiles == 32
  __syncwarp();
}

__device__ __forceinline__ void direct_count(uint32_t o, bool fin) {
  if (fin)
    atomicAdd(&direct_counts()[o >> kDirectShift], 1u);
}

__device__ __forceinline__ void direct_finish(const MLaunch& L) {
  const uint32_t lane = threadIdx.x & 31u;
  __syncwarp();
  const uint32_t mine = direct_counts()[lane];
  __threadfence();
  bool complete = false;
  if (mine) {
    const MTile& T = L.inl[lane];
    complete = atomicAdd(&L.tile_done[lane], mine) + mine == T.nrows * T.ncols;
  }
  uint32_t fins = __ballot_sync(kFull, complete);
  if (fins)
    __threadfence();
  while (fins) {
    const uint32_t t = (uint32_t)(__ffs(fins) - 1);
    fins &= fins - 1;
    const MTile& T = L.inl[t];
    const uint32_t nv = T.nrows * T.ncols / 4;
    CAFXG_DCHECK(t < L.n && (uint64_t)T.out_off + 4ull * nv <= L.out_limit &&
                 ((uintptr_t)T.reply & 15) == 0);
    const uint4* from = reinterpret_cast<const uint4*>(L.out + T.out_off);
    uint4* to = reinterpret_cast<uint4*>(T.reply);
    for (uint32_t i0 = 0; i0 < nv; i0 += 32 * 8) {
      uint4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t i = i0 + k * 32 + lane;
        if (i < nv)
          v[k] = __ldcg(from + i);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t i = i0 + k * 32 + lane;
        if (i < nv)
          to[i] = v[k];
      }
    }
    if (lane == t)
      L.tile_done[t] = 0;  // ready for the next launch on this staging slot
  }
}

// Self-resetting scheduler: the last block to finish zeroes the cursor so
// the slot can serve the next launch without a memset.
__device__ __forceinline__ void retire_block(const MLaunch& L) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    uint32_t prev = atomicAdd(&L.sched[1], 1u);
    if (prev == gridDim.x - 1) {
      L.sched[0] = 0;
      L.sched[1] = 0;
      __threadfence();
    }
  }
}

// ---- checked kernel: escape tested at every step ------------------------------
// 4 CTAs x 256 threads per SM (<= 64 registers): 8 warps per scheduler, each
// with two independent FP2 chains in fp32; fp64 is bound by the FP64 pipe.
// Used where the deferred kernel's precondition does not hold (tiles that
// reach |c| ~ 2) and for small max_iter.
// kMode 0: coordinates loaded from the tables of coords_kernel (big tiles);
// 1: computed at pixel start (batches of small tiles); 2: as 1, plus the
// direct reply (MLaunch::direct; 2 CTAs per SM so the copy path has
// registers).
template <class Slots, int kSteps, bool kExact, int kMode>
__global__ void __launch_bounds__(kMandelThreads, kMode == 2 ? 2 : 4)
    mandel_kernel(const __grid_constant__ MLaunch L) {
  constexpr bool kDirect = kMode == 2;
  constexpr int NS = Slots::kSlots;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t maxit = L.max_iter;  // uniform per launch
  constexpr uint32_t omask = kDirect ? (1u << kDirectShift) - 1u : 0xffffffffu;

  Feeder<Slots, kMode> feed;
  Slots sl;
  sl.zero = L.zero;
  uint32_t n[NS];   // iterations completed without escape; bit 31 = escaped
  uint32_t o[NS];   // output element offsets from L.out
  uint32_t live = 0;  // bit s: slot s holds a pixel
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    n[s] = 0;
    o[s] = 0;
  }

  if constexpr (kDirect)
    direct_begin();
  feed.refill(L, sl, n, o, live, lt_mask);
  while (__any_sync(kFull, live != 0)) {
    sl.template run<kSteps, kExact>(n);
    // escaped (bit 31) or reached max_iter; an escape at step i leaves i-1
    // non-escaped steps counted, so the reference's return value is n+1
    uint32_t done = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s)
      done |= ((live >> s & 1u) && n[s] >= maxit) ? (1u << s) : 0u;
    if (__any_sync(kFull, done != 0)) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (done >> s & 1u) {
          uint32_t c = (int32_t)n[s] < 0 ? (n[s] & 0x7fffffffu) + 1u : n[s];
          CAFXG_DCHECK((o[s] & omask) < L.out_limit);
          L.out[o[s] & omask] = min(c, maxit);
        }
      }
      if constexpr (kDirect) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
          direct_count(o[s], done >> s & 1u);
      }
      live &= ~done;
      feed.refill(L, sl, n, o, live, lt_mask);
    }
  }
  if constexpr (kDirect)
    direct_finish(L);
  retire_block(L);
}

// ---- deferred kernel: escape tested once per block ----------------------------
// The main loop runs kSteps iterations with no escape test at all (6 packed
// FP ops per pixel pair and step instead of 7 + FSETP + IADD), then tests
// fl(zr^2 + zi^2) > 4 (or NaN) once. A pixel that passes has not escaped in
// any of the kSteps steps; a pixel that fails is pushed -- with its z, c and
// count from the START of the block -- on a per-warp replay queue in shared
// memory and its slot is refilled. When the queue holds a full warp's worth
// (32 x kSlots entries) the warp replays those blocks with the checked
// per-step code, every lane busy; the replay evaluates the identical
// operation sequence from the identical state, so it finds the reference's
// escape step exactly.
//
// Why a block-end test sees every escape inside the block: once the reference
// test fires at step i, the orbit keeps |z| > 2 (and overflows to inf / NaN,
// which the unordered test also catches) for every later step, provided
// |c| <= 2 - eta or |c| >= 2 + eta with eta far above the rounding error
// (|z_{i+1}| >= |z_i|^2 - |c| > |z_i| + eta/2). The host runs this kernel only
// for tiles whose coordinate box stays outside 2 - 2^-10 < |c| < 2 + 2^-10
// (DESIGN.md §3.1); others take mandel_kernel. A block that crosses max_iter
// is handled the same way: no escape by the block end means none by max_iter,
// and a replayed pixel's count is clamped to max_iter as in mandel_kernel.
//
// 2 CTAs x 256 threads per SM: up to 128 registers, room for the replay
// slots next to the live ones; 4 warps x 2 chains per scheduler still keep
// the FP pipe saturated (6 FP2 ops of 2 cycles vs a 3-op dependency chain).
template <class Slots>
struct ReplayQueue {
  using Cd = typename Slots::C;
  static constexpr int kCap = 2 * 32 * Slots::kSlots;  // < 1 batch + 1 block of pushes
  Cd zr[kCap], zi[kCap], cr[kCap], ci[kCap];
  uint32_t n[kCap], o[kCap];
};

// Per warp: the replay queue and the mid-block checkpoint (the live slots'
// z after half a block; see mandel_deferred_kernel).
template <class Slots>
struct DeferredWarp {
  ReplayQueue<Slots> q;
  typename Slots::Mid mid;
};

template <class Slots>
constexpr size_t deferred_smem_bytes() {
  return sizeof(DeferredWarp<Slots>) * (kMandelThreads / 32);
}

// Replay window: the deferred kernel checkpoints z halfway through a fully
// unrolled block, so an escaped block replays at most half its steps (8-step
// units with runtime repeats keep whole-block replays).
__host__ __device__ constexpr int deferred_replay_steps(int unit) { return unit == 8 ? 8 : unit / 2; }

template <class Slots, int kUnit, bool kExact, bool kDirect>
__device__ __forceinline__ void replay(const MLaunch& L, ReplayQueue<Slots>& q,
                                       uint32_t first, uint32_t count, uint32_t maxit) {
  constexpr int NS = Slots::kSlots;
  const uint32_t lane = threadIdx.x & 31u;
  Slots rp;
  rp.zero = L.zero;
  uint32_t rn[NS], ro[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const uint32_t k = s * 32 + lane;
    if (k < count) {
      const uint32_t e = first + k;
      rp.resume(s, q.zr[e], q.zi[e], q.cr[e], q.ci[e]);
      rn[s] = q.n[e];
      ro[s] = q.o[e];
    } else {
      rp.start(s, 0, 0);  // c = 0 never escapes; result discarded
      rn[s] = 0;
      ro[s] = 0xffffffffu;
    }
  }
  __syncwarp();  // entries consumed before later pushes overwrite them
  if constexpr (kUnit == 8) {
#pragma unroll 1
    for (uint32_t r = 0; r < L.block_reps; ++r)
      rp.template run<kUnit, kExact>(rn);
  } else {
    rp.template run<deferred_replay_steps(kUnit), kExact>(rn);
  }
  constexpr uint32_t omask = kDirect ? (1u << kDirectShift) - 1u : 0xffffffffu;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (ro[s] != 0xffffffffu) {
      uint32_t c = (int32_t)rn[s] < 0 ? (rn[s] & 0x7fffffffu) + 1u : rn[s];
      CAFXG_DCHECK((ro[s] & omask) < L.out_limit);
      L.out[ro[s] & omask] = min(c, maxit);
    }
  }
  if constexpr (kDirect) {
#pragma unroll
    for (int s = 0; s < NS; ++s)
      direct_count(ro[s], ro[s] != 0xffffffffu);
  }
}

template <class Slots, int kUnit, bool kExact, int kMode>
__global__ void __launch_bounds__(kMandelThreads, 2)
    mandel_deferred_kernel(const __grid_constant__ MLaunch L) {
  constexpr bool kDirect = kMode == 2;
  constexpr int NS = Slots::kSlots;
  constexpr uint32_t kBatch = 32 * NS;
  using Cd = typename Slots::C;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DeferredWarp<Slots>& ws = reinterpret_cast<DeferredWarp<Slots>*>(smem_raw)[threadIdx.x >> 5];
  ReplayQueue<Slots>& q = ws.q;
  constexpr int kHalf = deferred_replay_steps(kUnit);
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t maxit = L.max_iter;
  // block length: kUnit unrolled steps x block_reps (chosen by the host so
  // that max_iter is (nearly) a multiple of it: no steps past max_iter)
  const uint32_t reps = L.block_reps;
  const uint32_t block = kUnit * reps;
  uint32_t* const out = L.out;
  constexpr uint32_t omask = kDirect ? (1u << kDirectShift) - 1u : 0xffffffffu;

  Feeder<Slots, kMode> feed;
  Slots sl;
  sl.zero = L.zero;
  uint32_t n[NS];  // steps completed (a multiple of the block), all unescaped
  uint32_t o[NS];
  uint32_t live = 0;
  uint32_t queued = 0;  // warp-uniform queue length
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    n[s] = 0;
    o[s] = 0;
  }

  if constexpr (kDirect)
    direct_begin();
  feed.refill(L, sl, n, o, live, lt_mask);
  while (__any_sync(kFull, live != 0)) {
    Cd szr[NS], szi[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      szr[s] = sl.zr_of(s);
      szi[s] = sl.zi_of(s);
    }
    if constexpr (kUnit == 8) {
#pragma unroll 1
      for (uint32_t r = 0; r < reps; ++r)
        sl.template run_free<kUnit, kExact>();
    } else {
      // fully unrolled block (the host sets block_reps = 1): no runtime loop,
      // which also spared ptxas a second copy of the block-start save. The
      // z halfway through goes to shared memory: an escaped block then
      // replays only the half its escape lies in.
      sl.template run_free<kHalf, kExact>();
      sl.save_mid(ws.mid, lane);
      sl.template run_free<kUnit - kHalf, kExact>();
    }
    const uint32_t esc = sl.escaped() & live;
    uint32_t done = esc;
    // counts first, then one rarely-taken branch for the stores (a pixel
    // reaches max_iter once in its lifetime): a store per slot compiled to
    // one BSSY region per slot, each re-loading max_iter and L.out
    const uint32_t blk = kUnit == 8 ? block : (uint32_t)kUnit;
    uint32_t hitm = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const bool act = ((live & ~esc) >> s) & 1u;
      n[s] += act ? blk : 0u;
      hitm |= (uint32_t)(act && n[s] >= maxit) << s;
    }
    if (hitm) {
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (hitm >> s & 1u) {
          CAFXG_DCHECK((o[s] & omask) < L.out_limit);
          out[o[s] & omask] = maxit;
        }
    }
    done |= hitm;
    if (__any_sync(kFull, esc != 0)) {
      uint32_t base = queued;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const uint32_t b = __ballot_sync(kFull, esc >> s & 1u);
        if (esc >> s & 1u) {
          const uint32_t e = base + __popc(b & lt_mask);
          Cd rz = szr[s], iz = szi[s];
          uint32_t rn = n[s];
          if constexpr (kUnit != 8) {
            // not yet escaped halfway (the orbit stays out once out, see
            // above): the escape lies in the second half
            const Cd mr = Slots::mid_zr(ws.mid, s, lane), mi = Slots::mid_zi(ws.mid, s, lane);
            if (!Slots::escaped_at(mr, mi)) {
              rz = mr;
              iz = mi;
              rn += kHalf;
            }
          }
          q.zr[e] = rz;
          q.zi[e] = iz;
          q.cr[e] = sl.cr_of(s);
          q.ci[e] = sl.ci_of(s);
          q.n[e] = rn;
          q.o[e] = o[s];
        }
        base += __popc(b);
      }
      queued = base;
    }
    if (__any_sync(kFull, done != 0)) {
      if constexpr (kDirect) {  // block-end finishes (escapes finish in replay)
#pragma unroll
        for (int s = 0; s < NS; ++s)
          direct_count(o[s], (done & ~esc) >> s & 1u);
      }
      live &= ~done;
      feed.refill(L, sl, n, o, live, lt_mask);
    }
    if (queued >= kBatch) {
      __syncwarp();
      queued -= kBatch;
      replay<Slots, kUnit, kExact, kDirect>(L, q, queued, kBatch, maxit);
    }
  }
  if (queued) {
    __syncwarp();
    replay<Slots, kUnit, kExact, kDirect>(L, q, 0, queued, maxit);
  }
  if constexpr (kDirect)
    direct_finish(L);
  retire_block(L);
}

template <class A, int kSteps, bool kExact>
int launch_t(const MLaunch& L, int grid, cudaStream_t s) {
  if (L.direct)
    mandel_kernel<A, kSteps, kExact, 2><<<grid, kMandelThreads, 0, s>>>(L);
  else if (L.inline_coords)
    mandel_kernel<A, kSteps, kExact, 1><<<grid, kMandelThreads, 0, s>>>(L);
  else
    mandel_kernel<A, kSteps, kExact, 0><<<grid, kMandelThreads, 0, s>>>(L);
  return (int)cudaGetLastError();
}

// Opts kernel `f` into `bytes` of dynamic shared memory on the current device
// (the attribute is per-device state: once per device and kernel).
template <class F>
cudaError_t opt_in_smem(F* f, size_t bytes, std::atomic<uint64_t>& done_mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && (done_mask.load(std::memory_order_acquire) >> dev & 1))
    return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && dev < 64)
    done_mask.fetch_or(1ull << dev);
  return e;
}

template <class A, int kUnit, bool kExact>
int launch_deferred_t(const MLaunch& L, int grid, cudaStream_t s) {
  constexpr size_t smem = deferred_smem_bytes<A>();
  if (L.direct) {
    // the direct-reply counters and the chunk coordinate tables (static
    // shared memory) push the kernel past the 48 KB that needs no opt-in
    static std::atomic<uint64_t> opted{0};
    if (cudaError_t e = opt_in_smem(mandel_deferred_kernel<A, kUnit, kExact, 2>, smem, opted))
      return (int)e;
    mandel_deferred_kernel<A, kUnit, kExact, 2><<<grid, kMandelThreads, smem, s>>>(L);
  } else if (L.inline_coords) {
    static std::atomic<uint64_t> opted{0};  // (the chunk coordinate tables, as above)
    if (cudaError_t e = opt_in_smem(mandel_deferred_kernel<A, kUnit, kExact, 1>, smem, opted))
      return (int)e;
    mandel_deferred_kernel<A, kUnit, kExact, 1><<<grid, kMandelThreads, smem, s>>>(L);
  } else {
    static std::atomic<uint64_t> opted{0};  // queues + checkpoints: > 48 KB
    if (cudaError_t e = opt_in_smem(mandel_deferred_kernel<A, kUnit, kExact, 0>, smem, opted))
      return (int)e;
    mandel_deferred_kernel<A, kUnit, kExact, 0><<<grid, kMandelThreads, smem, s>>>(L);
  }
  return (int)cudaGetLastError();
}

template <class A, int kSteps, bool kExact>
int occ_t() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, mandel_kernel<A, kSteps, kExact, 0>,
                                                kMandelThreads, 0);
  return n;
}

template <class A, int kUnit, bool kExact>
int occ_deferred_t() {
  static std::atomic<uint64_t> opted{0};
  opt_in_smem(mandel_deferred_kernel<A, kUnit, kExact, 0>, deferred_smem_bytes<A>(), opted);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &n, mandel_deferred_kernel<A, kUnit, kExact, 0>, kMandelThreads,
      deferred_smem_bytes<A>());
  return n;
}

// two CTAs per SM with their static chunk tables
static_assert(deferred_smem_bytes<F32Slots>() <= 96 * 1024, "replay queues exceed 96 KB");
static_assert(deferred_smem_bytes<F64Slots>() <= 96 * 1024, "replay queues exceed 96 KB");

}  // namespace

#define CAFXG_MANDEL_K(FN, SL, K, ...)                                 \
  return exact ? FN<SL, K, true>(__VA_ARGS__) : FN<SL, K, false>(__VA_ARGS__)
// checked kernel: ksteps 4 / 16 / 32 between refills
#define CAFXG_MANDEL_DISPATCH(FN, ...)                                 \
  do {                                                                 \
    if (precision == 0) {                                              \
      if (ksteps <= 4) CAFXG_MANDEL_K(FN, F32Slots, 4, __VA_ARGS__);   \
      if (ksteps <= 16) CAFXG_MANDEL_K(FN, F32Slots, 16, __VA_ARGS__); \
      CAFXG_MANDEL_K(FN, F32Slots, 32, __VA_ARGS__);                   \
    }                                                                  \
    if (ksteps <= 4) CAFXG_MANDEL_K(FN, F64Slots, 4, __VA_ARGS__);     \
    if (ksteps <= 16) CAFXG_MANDEL_K(FN, F64Slots, 16, __VA_ARGS__);   \
    CAFXG_MANDEL_K(FN, F64Slots, 32, __VA_ARGS__);                     \
  } while (0)
// deferred kernel: unrolled unit of 8 steps x runtime reps, or one
// fully unrolled 32-step block
#define CAFXG_DEFERRED_UNITS(FN, SL, ...)                              \
  do {                                                                 \
    if (unit == 8) CAFXG_MANDEL_K(FN, SL, 8, __VA_ARGS__);             \
    if (unit == 16) CAFXG_MANDEL_K(FN, SL, 16, __VA_ARGS__);           \
    if (unit == 24) CAFXG_MANDEL_K(FN, SL, 24, __VA_ARGS__);           \
    if (unit == 40) CAFXG_MANDEL_K(FN, SL, 40, __VA_ARGS__);           \
    if (unit == 48) CAFXG_MANDEL_K(FN, SL, 48, __VA_ARGS__);           \
    if (unit == 56) CAFXG_MANDEL_K(FN, SL, 56, __VA_ARGS__);           \
    if (unit == 64) CAFXG_MANDEL_K(FN, SL, 64, __VA_ARGS__);           \
    CAFXG_MANDEL_K(FN, SL, 32, __VA_ARGS__);                           \
  } while (0)
// deferred kernel: an unrolled unit of 16..48 steps (x block_reps, normally
// 1), or 8-step units x runtime reps for other block lengths
#define CAFXG_DEFERRED_DISPATCH(FN, ...)                               \
  do {                                                                 \
    if (precision == 0)                                                \
      CAFXG_DEFERRED_UNITS(FN, F32Slots, __VA_ARGS__);                 \
    CAFXG_DEFERRED_UNITS(FN, F64Slots, __VA_ARGS__);                   \
  } while (0)

int mandel_launch(const MLaunch& L0, int precision, const MandelLaunchCfg& cfg,
                  void* stream) {
  const bool exact = cfg.exact;
  cudaStream_t s = (cudaStream_t)stream;
  if (cfg.deferred) {
    const int unit = cfg.unit;
    MLaunch L = L0;
    L.block_reps = (uint32_t)cfg.reps;
    CAFXG_DEFERRED_DISPATCH(launch_deferred_t, L, cfg.grid, s);
  }
  const int ksteps = cfg.ksteps;
  CAFXG_MANDEL_DISPATCH(launch_t, L0, cfg.grid, s);
}

int mandel_coords_launch(const MLaunch& L, int precision, uint32_t max_extent,
                         void* stream) {
  if (L.n == 0)
    return 0;
  dim3 grid((max_extent + 255) / 256, L.n);
  if (grid.x > 64)
    grid.x = 64;
  if (precision == 0)
    coords_kernel<float><<<grid, 256, 0, (cudaStream_t)stream>>>(L);
  else
    coords_kernel<double><<<grid, 256, 0, (cudaStream_t)stream>>>(L);
  return (int)cudaGetLastError();
}

int mandel_max_blocks_per_sm(int precision, int ksteps, bool exact, bool deferred, int unit) {
  if (deferred)
    CAFXG_DEFERRED_DISPATCH(occ_deferred_t);
  CAFXG_MANDEL_DISPATCH(occ_t);
}

int mandel_slots_per_thread(int precision) {
  return precision == 0 ? F32Slots::kSlots : F64Slots::kSlots;
}

}  // namespace cafxg
