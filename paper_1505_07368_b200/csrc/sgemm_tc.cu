// 3xTF32 fp32 GEMM on the 5th-generation tensor cores (tcgen05) for the
// `matrix_multiply` compute actor: C = A * B, row-major.
//
// fp32 operands are split once per request into tf32 hi/lo halves
// (hi = rna_tf32(x), lo = rna_tf32(x - hi)); the kernel accumulates
// lo(A)*hi(B) + hi(A)*lo(B) + hi(A)*hi(B) in fp32 TMEM, which recovers ~22
// mantissa bits per product (the dropped lo*lo term is ~2^-22 relative).
//
// Kernel (one 128x256 C tile per CTA, 6 warps, warp-specialised):
//   warp 0 lane 0 : TMA producer -- 4-stage ring of {A_hi, A_lo, Bt_hi, Bt_lo}
//                   16-deep K slices (SWIZZLE_64B, K-major), mbarrier
//                   complete_tx;
//   warp 1        : allocates 512 TMEM columns (two 128x256 fp32
//                   accumulators); lane 0 issues tcgen05.mma.cta_group::1
//                   .kind::tf32 (M=128, N=256, K=8), 6 per stage, alternating
//                   accumulators every 128 K; tcgen05.commit frees stages and
//                   hands finished chunks to the epilogue;
//   warps 2..9    : epilogue -- tcgen05.ld 32x32b.x32 TMEM -> registers,
//                   fp32 round-to-nearest sum of the K chunks (the tensor
//                   core accumulates with truncation), then global stores
//                   (each thread owns half a C row of the tile).
// Grid: grouped raster over (M/128) x (N/256) tiles so the CTAs in flight
// share A row-blocks and B column-blocks in L2.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "sgemm.cuh"

namespace cafxg {
namespace {

constexpr int BM = 128, BK = 16, STAGES = 4;
constexpr int A_TILE = BM * BK * 4;                       // 8 KiB
constexpr int EPI_WARPS = 8;                              // 2 per TMEM lane quadrant
constexpr int TC_THREADS = 64 + EPI_WARPS * 32;           // TMA + MMA + epilogue
constexpr int GROUP_M = 16;  // default raster group (CAFXG_SGEMM_GROUP_M overrides)
// K chunk per accumulator: the tensor core's fp32 accumulation rounds toward
// zero, so its error grows linearly with the number of MMAs into one
// accumulator (measured: 3.9e-5 normwise at K=4096 with a single
// accumulator). Chunks of 128 K are summed by the epilogue in fp32 with
// round-to-nearest, which keeps the error at the per-chunk level.
constexpr int CHUNK_KB = 8;                               // k-blocks per chunk (128 K)
constexpr int kMaxSplits = 8;  // portable cluster size

// Tile width BN = 256 (large grids) or 128 (grids too small to fill the SMs:
// twice the CTAs per split-K factor, half the partial tile to reduce).
template <int BN>
struct Cfg {
  static constexpr int B_TILE = BN * BK * 4;                 // 16 / 8 KiB
  static constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;  // 48 / 32 KiB
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = 2 * BN;              // two BN-column accumulators
  static constexpr int COLS = BN / 2;                        // epilogue: half a tile row
  // Instruction descriptor: D=f32, A=B=tf32, K-major both, M=128, N=BN.
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  static_assert(BM * BN * 4 <= STAGES * STAGE_BYTES, "split-K partial must fit the stages");
};

// ---- PTX helpers -----------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// UMMA shared-memory descriptor, K-major SWIZZLE_64B canonical layout
// ((8,m),2):((4,SBO),1) in 16-byte units: 64-byte rows, 8-row groups 512 B
// apart (SBO), LBO unused (1), version 1 (sm_100), layout type 4.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;        // SBO
  d |= (uint64_t)1 << 46;                 // version
  d |= (uint64_t)4 << 61;                 // SWIZZLE_64B
  return d;
}

template <uint32_t IDESC>
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// split-K partial tile (128 x 256 fp32) in shared memory, float4 granules:
// row r, column granule c4 (0..63) XOR-swizzled by r % 8 so a warp storing
// one granule of 32 consecutive rows hits 8 distinct 16-byte bank groups
template <int BN>
__device__ __forceinline__ int partial_index(int r, int c4) {
  return r * (BN / 4) + (c4 ^ (r & 7));
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 16-byte load from the shared memory of cluster CTA `rank` at the address
// that `local` has in this CTA
__device__ __forceinline__ float4 ld_cluster_f4(uint32_t local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote)
               : "memory");
  return v;
}

// ---- the GEMM kernel --------------------------------------------------------

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    sgemm_3xtf32_kernel(const __grid_constant__ CUtensorMap mAh,
                        const __grid_constant__ CUtensorMap mAl,
                        const __grid_constant__ CUtensorMap mBh,
                        const __grid_constant__ CUtensorMap mBl, float* __restrict__ C,
                        int M, int N, int K, int ldc, int splits, int a_row0,
                        int b_row0, int group_m) {
  using G = Cfg<BN>;
  constexpr int STAGE_BYTES = G::STAGE_BYTES, B_TILE = G::B_TILE;
  // a_row0 / b_row0: first row of this GEMM's A / B^T block inside the
  // matrices the tensor maps describe (a sub-block of a larger product)
  // split-K: the `splits` CTAs of one C tile form a thread-block cluster; CTA
  // z covers K range [z*K/splits, (z+1)*K/splits), parks its partial tile in
  // its own shared memory, and after a cluster barrier each CTA sums 1/splits
  // of the tile's rows over the peers' partials through distributed shared
  // memory, in fixed z order (deterministic; no workspace, no extra launch)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;    // [2] chunk accumulated (MMA -> epilogue)
  uint64_t* acc_empty = acc_full + 2;     // [2] chunk consumed (epilogue -> MMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // grouped raster: GROUP_M consecutive M tiles share each N tile
  const int tiles_m = M / BM, tiles_n = N / BN;
  const int per_group = group_m * tiles_n;
  const int kz = blockIdx.x % splits;   // == %cluster_ctarank (cluster = splits x 1 x 1)
  const int bid = blockIdx.x / splits;
  const int first_m = (bid / per_group) * group_m;
  const int gsize = min(group_m, tiles_m - first_m);
  const int in_group = bid % per_group;
  const int m0 = (first_m + in_group % gsize) * BM;
  const int n0 = (in_group / gsize) * BN;
  const int ksplit = K / splits;
  const int k_base = kz * ksplit;
  const int nk = ksplit / BK;

  if (warp == 0 && lane == 0) {
    for (const CUtensorMap* m : {&mAh, &mAl, &mBh, &mBl})
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m))
                   : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(G::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: everything above (barrier init, TMEM
  // allocation, tensor-map prefetch) overlaps the tail of the operand split;
  // no global memory is touched before the split grid has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* st = smem + s * STAGE_BYTES;
      mbar_expect_tx(&full[s], STAGE_BYTES);
      const int kx = k_base + kb * BK;
      tma_load_2d(st, &mAh, &full[s], kx, a_row0 + m0);
      tma_load_2d(st + A_TILE, &mAl, &full[s], kx, a_row0 + m0);
      tma_load_2d(st + 2 * A_TILE, &mBh, &full[s], kx, b_row0 + n0);
      tma_load_2d(st + 2 * A_TILE + B_TILE, &mBl, &full[s], kx, b_row0 + n0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer ----
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      const int chunk = kb / CHUNK_KB, kin = kb % CHUNK_KB;
      const uint32_t acc = tmem + (uint32_t)(chunk & 1) * BN;
      if (kin == 0)  // the epilogue must have drained this accumulator
        mbar_wait(&acc_empty[chunk & 1], ((chunk >> 1) & 1) ^ 1);
      mbar_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
      const uint32_t ah = base, al = base + A_TILE;
      const uint32_t bh = base + 2 * A_TILE, bl = bh + B_TILE;
#pragma unroll
      for (int k = 0; k < BK / 8; ++k) {
        const uint32_t off = k * 32;  // 8 tf32 = 32 bytes along K
        const uint32_t acc0 = (kin | k) != 0;
        mma_tf32<G::IDESC>(acc, umma_desc_sw64(al + off), umma_desc_sw64(bh + off), acc0);
        mma_tf32<G::IDESC>(acc, umma_desc_sw64(ah + off), umma_desc_sw64(bl + off), 1);
        mma_tf32<G::IDESC>(acc, umma_desc_sw64(ah + off), umma_desc_sw64(bh + off), 1);
      }
      umma_commit(&empty[s]);  // the stage is free once these MMAs retire
      if (kin == CHUNK_KB - 1 || kb == nk - 1)
        umma_commit(&acc_full[chunk & 1]);
    }
  } else if (warp >= 2) {
    // ---- epilogue: sum the chunk accumulators in fp32 (RN), then store ----
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;       // which half of the tile's columns
    const int row = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    float sum[G::COLS];
#pragma unroll
    for (int j = 0; j < G::COLS; ++j)
      sum[j] = 0.0f;
    const int nchunks = (nk + CHUNK_KB - 1) / CHUNK_KB;
    for (int chunk = 0; chunk < nchunks; ++chunk) {
      const int b = chunk & 1;
      mbar_wait(&acc_full[b], (chunk >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int c = 0; c < G::COLS / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + (uint32_t)(b * BN + half * G::COLS + c * 32), r);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          sum[c * 32 + j] = __fadd_rn(sum[c * 32 + j], __uint_as_float(r[j]));
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&acc_empty[b]))
                     : "memory");
    }
    if (splits == 1) {
      float* crow = C + (size_t)(m0 + row) * ldc + n0 + half * G::COLS;
#pragma unroll
      for (int j = 0; j < G::COLS; j += 4)
        *reinterpret_cast<float4*>(crow + j) =
            make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]);
    } else {
      // partial tile into the (now idle) stage buffers: the last acc_full
      // commit follows every MMA, so no TMA write or MMA read is pending
      float4* part = reinterpret_cast<float4*>(smem);
#pragma unroll
      for (int j = 0; j < G::COLS; j += 4)
        part[partial_index<BN>(row, half * (G::COLS / 4) + j / 4)] =
            make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (splits > 1) {
    cluster_sync();  // every partial of the cluster is written
    const int rows = BM / splits;
    const uint32_t mine = smem_u32(smem);
    for (int i = threadIdx.x; i < rows * (BN / 4); i += TC_THREADS) {
      const int r = kz * rows + i / (BN / 4), c4 = i % (BN / 4);
      const uint32_t off = (uint32_t)partial_index<BN>(r, c4) * 16u;
      float4 acc = ld_cluster_f4(mine + off, 0);
      for (int z = 1; z < splits; ++z) {
        const float4 v = ld_cluster_f4(mine + off, (uint32_t)z);
        acc.x = __fadd_rn(acc.x, v.x);
        acc.y = __fadd_rn(acc.y, v.y);
        acc.z = __fadd_rn(acc.z, v.z);
        acc.w = __fadd_rn(acc.w, v.w);
      }
      *reinterpret_cast<float4*>(C + (size_t)(m0 + r) * ldc + n0 + c4 * 4) = acc;
    }
    cluster_sync();  // the peers are done reading this CTA's partial
  }
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(G::TMEM_COLS));
}

// ---- hi/lo split ----------------------------------------------------------

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  float rest = __fsub_rn(x, hi);  // exact
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(rest));
  lo = __uint_as_float(l);
}

// A (M x K, lda) -> Ah, Al (M x K packed)
__global__ void __launch_bounds__(256) split_rows_kernel(const float* __restrict__ A, int lda,
                                                         int M, int K, float* __restrict__ Ah,
                                                         float* __restrict__ Al) {
  const size_t total = (size_t)M * K;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total / 4;
       i += (size_t)gridDim.x * blockDim.x) {
    size_t e = i * 4;
    size_t r = e / K, c = e % K;
    float4 v = *reinterpret_cast<const float4*>(A + r * lda + c);
    float4 h, l;
    split_tf32(v.x, h.x, l.x);
    split_tf32(v.y, h.y, l.y);
    split_tf32(v.z, h.z, l.z);
    split_tf32(v.w, h.w, l.w);
    *reinterpret_cast<float4*>(Ah + e) = h;
    *reinterpret_cast<float4*>(Al + e) = l;
  }
  asm volatile("griddepcontrol.launch_dependents;");
}

// B (K x N, ldb) -> Bth, Btl (N x K packed): 32x32 tiles through smem
__global__ void __launch_bounds__(256) split_transpose_kernel(const float* __restrict__ B,
                                                              int ldb, int K, int N,
                                                              float* __restrict__ Bth,
                                                              float* __restrict__ Btl) {
  __shared__ float th[32][33], tl[32][33];
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int j = ty; j < 32; j += 8) {
    float h, l;
    split_tf32(B[(size_t)(k0 + j) * ldb + n0 + tx], h, l);
    th[j][tx] = h;
    tl[j][tx] = l;
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    Bth[(size_t)(n0 + j) * K + k0 + tx] = th[tx][j];
    Btl[(size_t)(n0 + j) * K + k0 + tx] = tl[tx][j];
  }
  asm volatile("griddepcontrol.launch_dependents;");
}

// Both operands in one launch (device-API requests): blocks [0, nb_a) split
// A's rows, the rest split + transpose 64 x 64 tiles of B (K % 64 == 0).
__global__ void __launch_bounds__(256) split_ab_kernel(const float* __restrict__ A, int lda,
                                                       int M, int K, float* __restrict__ Ah,
                                                       float* __restrict__ Al,
                                                       const float* __restrict__ B, int ldb,
                                                       int N, float* __restrict__ Bth,
                                                       float* __restrict__ Btl, int nb_a) {
  if ((int)blockIdx.x < nb_a) {
    // rows of A in float4 steps; 32-bit index math (sgemm_tc_launch checks
    // M * K / 4 < 2^32)
    const uint32_t k4 = (uint32_t)K / 4, total = (uint32_t)M * k4;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint32_t)nb_a * blockDim.x) {
      const uint32_t r = i / k4, c = (i - r * k4) * 4;
      float4 v = *reinterpret_cast<const float4*>(A + (size_t)r * lda + c);
      float4 h, l;
      split_tf32(v.x, h.x, l.x);
      split_tf32(v.y, h.y, l.y);
      split_tf32(v.z, h.z, l.z);
      split_tf32(v.w, h.w, l.w);
      *reinterpret_cast<float4*>(Ah + (size_t)i * 4) = h;
      *reinterpret_cast<float4*>(Al + (size_t)i * 4) = l;
    }
    asm volatile("griddepcontrol.launch_dependents;");
    return;
  }
  // B: 64 x 64 tiles of (k, n), float4 loads along n and float4 stores
  // along k of the transposed halves (16-byte accesses both ways; 64 x 65
  // shared tiles keep the column reads conflict-free)
  __shared__ float th[64][65], tl[64][65];
  const int t = (int)blockIdx.x - nb_a, tn = N / 64;
  const int k0 = (t / tn) * 64, n0 = (t % tn) * 64;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = threadIdx.x + i * 256;          // float4 index in the 64 x 16 grid
    const int kk = f >> 4, nn = (f & 15) * 4;
    const float4 v = *reinterpret_cast<const float4*>(B + (size_t)(k0 + kk) * ldb + n0 + nn);
    float h, l;
    split_tf32(v.x, h, l); th[kk][nn + 0] = h; tl[kk][nn + 0] = l;
    split_tf32(v.y, h, l); th[kk][nn + 1] = h; tl[kk][nn + 1] = l;
    split_tf32(v.z, h, l); th[kk][nn + 2] = h; tl[kk][nn + 2] = l;
    split_tf32(v.w, h, l); th[kk][nn + 3] = h; tl[kk][nn + 3] = l;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = threadIdx.x + i * 256;          // float4 index in the 64 (n) x 16 (k) grid
    const int nn = f >> 4, kk = (f & 15) * 4;
    const float4 h = make_float4(th[kk][nn], th[kk + 1][nn], th[kk + 2][nn], th[kk + 3][nn]);
    const float4 l = make_float4(tl[kk][nn], tl[kk + 1][nn], tl[kk + 2][nn], tl[kk + 3][nn]);
    *reinterpret_cast<float4*>(Bth + (size_t)(n0 + nn) * K + k0 + kk) = h;
    *reinterpret_cast<float4*>(Btl + (size_t)(n0 + nn) * K + k0 + kk) = l;
  }
  asm volatile("griddepcontrol.launch_dependents;");
}

// The same with 32 x 32 tiles of B (K not a multiple of 64).
__global__ void __launch_bounds__(256) split_ab32_kernel(const float* __restrict__ A, int lda,
                                                       int M, int K, float* __restrict__ Ah,
                                                       float* __restrict__ Al,
                                                       const float* __restrict__ B, int ldb,
                                                       int N, float* __restrict__ Bth,
                                                       float* __restrict__ Btl, int nb_a) {
  __shared__ float th[32][33], tl[32][33];
  if ((int)blockIdx.x < nb_a) {
    // rows of A in float4 steps; 32-bit index math (sgemm_tc_launch checks
    // M * K / 4 < 2^32)
    const uint32_t k4 = (uint32_t)K / 4, total = (uint32_t)M * k4;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint32_t)nb_a * blockDim.x) {
      const uint32_t r = i / k4, c = (i - r * k4) * 4;
      float4 v = *reinterpret_cast<const float4*>(A + (size_t)r * lda + c);
      float4 h, l;
      split_tf32(v.x, h.x, l.x);
      split_tf32(v.y, h.y, l.y);
      split_tf32(v.z, h.z, l.z);
      split_tf32(v.w, h.w, l.w);
      *reinterpret_cast<float4*>(Ah + (size_t)i * 4) = h;
      *reinterpret_cast<float4*>(Al + (size_t)i * 4) = l;
    }
    asm volatile("griddepcontrol.launch_dependents;");
    return;
  }
  const int t = (int)blockIdx.x - nb_a, tn = N / 32;
  const int k0 = (t / tn) * 32, n0 = (t % tn) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int j = ty; j < 32; j += 8) {
    float h, l;
    split_tf32(B[(size_t)(k0 + j) * ldb + n0 + tx], h, l);
    th[j][tx] = h;
    tl[j][tx] = l;
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    Bth[(size_t)(n0 + j) * K + k0 + tx] = th[tx][j];
    Btl[(size_t)(n0 + j) * K + k0 + tx] = tl[tx][j];
  }
  asm volatile("griddepcontrol.launch_dependents;");
}

// ---- tensor maps (driver entry point fetched through the runtime) ---------

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled get_encoder() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

// rows x cols fp32 row-major (cols contiguous); box = box_rows x BK
bool make_map(CUtensorMap* m, const float* base, int rows, int cols, int box_rows) {
  EncodeTiled enc = get_encoder();
  if (!enc)
    return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool sgemm_tc_supported(int M, int N, int K, int lda, int ldb, int ldc) {
  (void)ldb;
  return M >= BM && N >= 128 && K >= BK && M % BM == 0 && N % 128 == 0 && K % 32 == 0 &&
         lda % 4 == 0 && ldc % 4 == 0 && get_encoder() != nullptr;
}

size_t sgemm_tc_scratch_bytes(int M, int N, int K) {
  // hi/lo splits of A and B^T (split-K reduces through distributed shared
  // memory and needs no workspace)
  return ((size_t)M * K * 2 + (size_t)N * K * 2) * sizeof(float);
}

int sgemm_tc_split_a(const float* A, int lda, int M, int K, float* Ah, float* Al,
                     void* stream) {
  int grid = (int)std::min<size_t>(((size_t)M * K / 4 + 255) / 256, 148 * 16);
  if (grid > 0)
    split_rows_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A, lda, M, K, Ah, Al);
  return (int)cudaGetLastError();
}

int sgemm_tc_split_b(const float* B, int ldb, int K, int N, float* Bh, float* Bl,
                     void* stream) {
  split_transpose_kernel<<<dim3(N / 32, K / 32), 256, 0, (cudaStream_t)stream>>>(B, ldb, K, N,
                                                                                Bh, Bl);
  return (int)cudaGetLastError();
}

namespace {

template <int BN>
void configure_once() {
  // once per device (the attribute is per-device state)
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !(configured.load() >> dev & 1)) {
    cudaFuncSetAttribute(sgemm_3xtf32_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Cfg<BN>::SMEM_BYTES);
    configured.fetch_or(1ull << dev);
  }
}

// How many clusters of `splits` CTAs of the GEMM kernel can be resident at
// once (clusters are placed within one GPC / die, so this is less than
// sms / splits: e.g. 8-CTA clusters do not all fit 148 SMs).
template <int BN>
int max_active_clusters(int splits) {
  static std::atomic<int> cache[kMaxSplits + 1];
  int v = cache[splits].load();
  if (v)
    return v;
  configure_once<BN>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(splits * 256));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = Cfg<BN>::SMEM_BYTES;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, sgemm_3xtf32_kernel<BN>, &cfg) != cudaSuccess ||
      n < 1) {
    cudaGetLastError();
    n = 148 / splits;
  }
  cache[splits].store(n);
  return n;
}

// CAFXG_SGEMM_PDL=0 launches the GEMM without programmatic dependent launch
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_SGEMM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int BN>
int launch(const CUtensorMap* m, float* C, int M, int N, int K, int ldc, void* stream,
           int splits, int a_row0, int b_row0) {
  configure_once<BN>();
  if (splits < 1 || splits > kMaxSplits || (splits & (splits - 1)) ||
      K % (16 * splits) != 0)
    splits = 1;
  const int tiles = (M / BM) * (N / BN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(tiles * splits));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = Cfg<BN>::SMEM_BYTES;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch (the kernel waits with griddepcontrol.wait
  // before touching global memory, so any predecessor is safe)
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  static const int group_m = [] {
    const char* e = getenv("CAFXG_SGEMM_GROUP_M");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : GROUP_M;
  }();
  cudaLaunchKernelEx(&cfg, sgemm_3xtf32_kernel<BN>, m[0], m[1], m[2], m[3], C, M, N, K, ldc,
                     splits, a_row0, b_row0, group_m);
  return (int)cudaGetLastError();
}

}  // namespace

// Tile width: 256 columns; 128 only for N a multiple of 128 but not 256. (A
// 128-column tile halves the split-K partial a cluster reduces, but each of
// its MMAs reads as much A as a 256-column one for half the work: at 1024^3
// with split-K 2 it measured 36.0 us against 34.6 us for 256 columns with
// split-K 4, and 2048^3 0.140 against 0.102 ms.) CAFXG_SGEMM_BN=128 forces
// the narrow tile (experiments).
int sgemm_tc_pick_bn(int M, int N, int sms) {
  (void)M;
  (void)sms;
  static const int env = [] {
    const char* e = getenv("CAFXG_SGEMM_BN");
    return e ? atoi(e) : 0;
  }();
  if (N % 256 != 0 || env == 128)
    return 128;
  return 256;
}

// Split-K factor (thread-block cluster size) for C grids too small to fill
// the GPU: the largest power of two <= 8 whose clusters (one per C tile) are
// all resident at once and that keeps every split >= 128 deep in K (one
// accumulator chunk).
int sgemm_tc_splits(int M, int N, int K, int sms, int bn) {
  (void)sms;
  const int tiles = (M / BM) * (N / bn);
  int s = 1;
  while (s < kMaxSplits && K % (16 * s * 2) == 0 && K / (s * 2) >= 128 &&
         tiles <= (bn == 256 ? max_active_clusters<256>(s * 2)
                             : max_active_clusters<128>(s * 2)))
    s *= 2;
  return s;
}

int sgemm_tc_make_maps(const float* Ah, const float* Al, int a_rows, const float* Bh,
                       const float* Bl, int N, int K, int bn, SgemmTcMaps* maps) {
  static_assert(sizeof(CUtensorMap) <= sizeof(maps->m[0]), "tensor map storage");
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(maps->m);
  maps->bn = bn;
  if (!make_map(&m[0], Ah, a_rows, K, BM) || !make_map(&m[1], Al, a_rows, K, BM) ||
      !make_map(&m[2], Bh, N, K, bn) || !make_map(&m[3], Bl, N, K, bn))
    return (int)cudaErrorInvalidValue;
  return 0;
}

int sgemm_tc_gemm_maps(const SgemmTcMaps* maps, float* C, int M, int N, int K, int ldc,
                       void* stream, int splits, int a_row0, int b_row0) {
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps->m);
  if (maps->bn == 256)
    return launch<256>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0);
  return launch<128>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0);
}

int sgemm_tc_gemm(const float* Ah, const float* Al, const float* Bh, const float* Bl, float* C,
                  int M, int N, int K, int ldc, void* stream, int splits, int bn) {
  SgemmTcMaps maps;
  if (int e = sgemm_tc_make_maps(Ah, Al, M, Bh, Bl, N, K, bn, &maps))
    return e;
  return sgemm_tc_gemm_maps(&maps, C, M, N, K, ldc, stream, splits);
}

int sgemm_tc_launch(const float* A, const float* B, float* C, int M, int N, int K, int lda,
                    int ldb, int ldc, void* scratch, int sm_count, void* stream,
                    int* launches, int splits_req) {
  float* Ah = static_cast<float*>(scratch);
  float* Al = Ah + (size_t)M * K;
  float* Bh = Al + (size_t)M * K;
  float* Bl = Bh + (size_t)N * K;
  if ((size_t)M * K / 4 >= (1ull << 32))
    return (int)cudaErrorInvalidValue;
  const int sms = sm_count > 0 ? sm_count : 148;
  const int bn = sgemm_tc_pick_bn(M, N, sms);
  const int splits = splits_req > 0 ? splits_req : sgemm_tc_splits(M, N, K, sms, bn);
  const int nb_a = (int)std::min<size_t>(((size_t)M * K / 4 + 255) / 256, 148 * 8);
  if (K % 64 == 0 && ldb % 4 == 0 && ((uintptr_t)B & 15) == 0) {
    const int nb_b = (N / 64) * (K / 64);
    split_ab_kernel<<<nb_a + nb_b, 256, 0, (cudaStream_t)stream>>>(A, lda, M, K, Ah, Al, B,
                                                                   ldb, N, Bh, Bl, nb_a);
  } else {
    const int nb_b = (N / 32) * (K / 32);
    split_ab32_kernel<<<nb_a + nb_b, 256, 0, (cudaStream_t)stream>>>(A, lda, M, K, Ah, Al, B,
                                                                     ldb, N, Bh, Bl, nb_a);
  }
  int e = (int)cudaGetLastError();
  if (e == 0)
    e = sgemm_tc_gemm(Ah, Al, Bh, Bl, C, M, N, K, ldc, stream, splits, bn);
  if (launches)
    *launches = 2;
  return e;
}

}  // namespace cafxg
