// 3xTF32 fp32 GEMM on the 5th-generation tensor cores (tcgen05) for the
// `matrix_multiply` compute actor: C = A * B, row-major.
//
// Each operand is taken as hi + lo tf32 halves and the kernel accumulates
// lo(A)*hi(B) + hi(A)*lo(B) + hi(A)*hi(B) in fp32 TMEM (~22 mantissa bits
// per product). Two operand forms, chosen per request by size:
//   split:  a pass writes hi = rna_tf32(x), lo = rna_tf32(x - hi) of A and of
//           B transposed (B^T, K-major); large GEMMs, where the pass is
//           cheap against the GEMM and K-major B feeds the MMA fastest;
//   raw:    the tensor core reads a 32-bit operand as tf32 by dropping its
//           low 13 mantissa bits, so A and B themselves are the hi halves;
//           a pass writes only lo = rna_tf32(x - trunc_tf32(x)), in place
//           layout (B stays K x N, an MN-major operand): half the pass's
//           writes, no transpose; small and mid-size GEMMs.
//
// Kernel (one 128 x BN C tile per CTA, BN = 256 or 128, 10 warps,
// warp-specialised):
//   warp 0 lane 0 : TMA producer -- 4-stage ring of {A_hi, A_lo, B_hi, B_lo}
//                   16-deep K slices (A and B^T K-major SWIZZLE_64B; raw B
//                   MN-major SWIZZLE_128B_ATOM_32B, one 3-D box per half),
//                   mbarrier complete_tx;
//   warp 1        : allocates 2 * BN TMEM columns (two 128 x BN fp32
//                   accumulators); lane 0 issues tcgen05.mma.cta_group::1
//                   .kind::tf32 (M=128, N=BN, K=8), 6 per stage, alternating
//                   accumulators every 128 K; tcgen05.commit frees stages and
//                   hands finished chunks to the epilogue;
//   warps 2..9    : epilogue -- tcgen05.ld 32x32b.x32 TMEM -> registers,
//                   fp32 round-to-nearest sum of the K chunks (the tensor
//                   core accumulates with truncation), then global stores
//                   (each thread owns half a C row of the tile).
// Grid: grouped raster over (M/128) x (N/BN) tiles so the CTAs in flight
// share A row-blocks and B column-blocks in L2. Grids too small to fill the
// GPU split K over a thread-block cluster; the partial tiles are reduced
// through an L2 workspace (device-API requests) or distributed shared memory.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "dcheck.cuh"
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
template <int BN, bool BMN>
struct Cfg {
  static constexpr int B_TILE = BN * BK * 4;                 // 16 / 8 KiB
  static constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;  // 48 / 32 KiB
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = 2 * BN;              // two BN-column accumulators
  static constexpr int COLS = BN / 2;                        // epilogue: half a tile row
  // Instruction descriptor: D=f32, A=B=tf32, A K-major, B K-major (B^T
  // split operands) or MN-major (BMN: raw B and its lo half), M=128, N=BN.
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    ((BMN ? 1u : 0u) << 16) |
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

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
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

// UMMA descriptor of an MN-major B operand (B as it lies in memory: K rows
// of N contiguous floats; no transpose). For 32-bit (tf32) MN-major operands
// the tensor core takes only the SWIZZLE_128B_BASE32B layout (type 1):
// 128-byte rows of 32 consecutive N columns with 32-byte granules XOR-ed by
// the row inside 4-row (512 B) atoms, which TMA writes with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B. A stage holds BN / 32 such 32-column
// chunks of BK rows, B_CHUNK bytes apart (LBO); 4-row K atoms are 512 B
// apart (SBO); one MMA of K = 8 spans two atoms (1024 B). (With the plain
// SWIZZLE_128B layout the MMA returns zeros.)
constexpr int B_CHUNK = 32 * BK * 4;  // 32 columns x BK rows: 2 KiB
__device__ __forceinline__ uint64_t umma_desc_mn_sw128b32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(B_CHUNK >> 4) << 16;  // LBO: next 32 N columns
  d |= (uint64_t)(512 >> 4) << 32;      // SBO: next 4 K rows
  d |= (uint64_t)1 << 46;               // version
  d |= (uint64_t)1 << 61;               // SWIZZLE_128B_BASE32B
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

// address in the shared memory of cluster CTA `rank` of the byte that
// `local` addresses in this CTA (windows are linear: offsets carry over)
__device__ __forceinline__ uint32_t cluster_map(uint32_t local, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  return remote;
}

// 16-byte distributed-shared-memory load (no memory clobber: the cluster
// barriers around the reduction order it against the partials' stores;
// volatile keeps the issue order the reduction loop writes)
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t remote) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote));
  return v;
}

// Phase timestamps for tuning (build with -DCAFXG_SGEMM_PHASES, `make
// phases`; tools/sgemm_phases.py reads them): %globaltimer per CTA at fixed
// points of the kernel, and the first start / last end of the split pass.
#ifdef CAFXG_SGEMM_PHASES
__device__ unsigned long long g_sgemm_phase[1024][16];  // [0, 8) globaltimer, [8, 16) clock64
__device__ unsigned long long g_split_span[2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SGEMM_PHASE(i)                                   \
  do {                                                   \
    if (blockIdx.x < 1024) {                             \
      g_sgemm_phase[blockIdx.x][i] = gtimer();           \
      g_sgemm_phase[blockIdx.x][8 + i] = clock64();      \
    }                                                    \
  } while (0)
#define SPLIT_SPAN_BEGIN() \
  if (threadIdx.x == 0) atomicMin(&g_split_span[0], gtimer())
#define SPLIT_SPAN_END()  \
  __syncthreads();        \
  if (threadIdx.x == 0) atomicMax(&g_split_span[1], gtimer())
#else
#define SGEMM_PHASE(i) \
  do {                 \
  } while (0)
#define SPLIT_SPAN_BEGIN()
#define SPLIT_SPAN_END()
#endif

// Split-K reduction through L2 (S = splits): this CTA (rank kz of cluster
// `bid`) sums rows [kz * BM / S, (kz + 1) * BM / S) of its tile over its own
// parked partial (shared memory) and the S - 1 slices its peers wrote to the
// workspace, in fixed z order. Every load of a thread's batch of granules is
// issued before the first add: the loop is L2-latency-bound otherwise.
template <int BN, int S>
__device__ __forceinline__ void reduce_ws(const float* __restrict__ ws, const uint8_t* smem,
                                          int bid, int kz, float* __restrict__ ctile, int ldc) {
  constexpr int ROWS = BM / S, N4 = ROWS * (BN / 4), PER = 4;
  const float4* mine = reinterpret_cast<const float4*>(ws) + ((size_t)bid * S + kz) * S * N4;
  for (int i0 = threadIdx.x; i0 < N4; i0 += PER * TC_THREADS) {
    float4 v[PER][S];
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int i = i0 + p * TC_THREADS;
#pragma unroll
      for (int z = 0; z < S; ++z)
        if (i < N4 && z != kz)
          v[p][z] = __ldcg(mine + (size_t)z * N4 + i);
    }
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int i = i0 + p * TC_THREADS;
      if (i >= N4)
        break;
      const int j4 = i / ROWS, rr = i - j4 * ROWS;
      const float4 l = *reinterpret_cast<const float4*>(
          smem + (uint32_t)partial_index<BN>(kz * ROWS + rr, j4) * 16u);
      float4 a = kz == 0 ? l : v[p][0];
#pragma unroll
      for (int z = 1; z < S; ++z) {
        const float4 w = z == kz ? l : v[p][z];
        a.x = __fadd_rn(a.x, w.x);
        a.y = __fadd_rn(a.y, w.y);
        a.z = __fadd_rn(a.z, w.z);
        a.w = __fadd_rn(a.w, w.w);
      }
      *reinterpret_cast<float4*>(ctile + (size_t)(kz * ROWS + rr) * ldc + j4 * 4) = a;
    }
  }
}

// ---- the GEMM kernel --------------------------------------------------------

// Where the 1-SM kernel's B stages come from. OneB: one (hi, lo) pair of
// tensor maps over the whole of B (or B^T). PeerBLoad (the multi-device fused
// path): one pair per K slice, each slice resident in the memory of the
// device that uploaded it; the producer picks the slice of each k-block, so
// the TMA engine pulls remote slices over NVLink tile by tile as the MMAs
// consume them -- the all-gather of B becomes the GEMM's own loads.
struct OneB {
  const CUtensorMap* h;
  const CUtensorMap* l;
  __device__ __forceinline__ void prefetch() const {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(h)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(l)) : "memory");
  }
  template <bool BMN>
  __device__ __forceinline__ void load(uint8_t* dh, uint8_t* dl, uint64_t* bar, int kx,
                                       int ncol) const {
    if constexpr (BMN) {
      // (one 3-D box: 32 columns x BK rows x BN / 32 chunks)
      tma_load_3d(dh, h, bar, 0, kx, ncol / 32);
      tma_load_3d(dl, l, bar, 0, kx, ncol / 32);
    } else {
      tma_load_2d(dh, h, bar, kx, ncol);
      tma_load_2d(dl, l, bar, kx, ncol);
    }
  }
};

constexpr int kMaxPeerSlices = 8;
struct PeerB {
  CUtensorMap h[kMaxPeerSlices], l[kMaxPeerSlices];  // raw B / lo(B), MN-major
  int kslice;                                          // K rows per slice
  int n;                                               // slices
};

struct PeerBLoad {
  const PeerB* p;
  __device__ __forceinline__ void prefetch() const {
    for (int i = 0; i < p->n; ++i) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p->h[i]))
                   : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p->l[i]))
                   : "memory");
    }
  }
  template <bool BMN>
  __device__ __forceinline__ void load(uint8_t* dh, uint8_t* dl, uint64_t* bar, int kx,
                                       int ncol) const {
    static_assert(BMN, "peer slices are raw MN-major B");
    const int src = kx / p->kslice, k = kx - src * p->kslice;
    CAFXG_DCHECK(src < p->n && k + BK <= p->kslice);
    tma_load_3d(dh, &p->h[src], bar, 0, k, ncol / 32);
    tma_load_3d(dl, &p->l[src], bar, 0, k, ncol / 32);
  }
};

template <int BN, bool BMN, class BSrc>
__device__ __forceinline__ void gemm_body(const CUtensorMap& mAh, const CUtensorMap& mAl,
                                          const BSrc& bsrc, float* __restrict__ C, int M,
                                          int N, int K, int ldc, int splits, int a_row0,
                                          int b_row0, int group_m, float* __restrict__ ws) {
  using G = Cfg<BN, BMN>;
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
  if (threadIdx.x == 0)
    SGEMM_PHASE(0);

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
  CAFXG_DCHECK(bid < tiles_m * tiles_n && m0 + BM <= M && n0 + BN <= N && nk > 0 &&
               ksplit % BK == 0);

  if (warp == 0 && lane == 0) {
    for (const CUtensorMap* m : {&mAh, &mAl})
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m))
                   : "memory");
    bsrc.prefetch();
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
  if (threadIdx.x == 0)
    SGEMM_PHASE(1);

  // Roles are warp-uniform branches (lane 0 works, the warp waits at
  // __syncwarp): the __syncthreads below is bar.sync, which PTX defines only
  // for warps that reach it converged.
  if (warp == 0) {
    // ---- TMA producer ----
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        const int kx = k_base + kb * BK;
        tma_load_2d(st, &mAh, &full[s], kx, a_row0 + m0);
        tma_load_2d(st + A_TILE, &mAl, &full[s], kx, a_row0 + m0);
        // B^T rows, or (BMN) raw B and its lo half as they lie (K rows of N
        // floats, BN / 32 chunks of 32 columns; b_row0 is then the first column)
        bsrc.template load<BMN>(st + 2 * A_TILE, st + 2 * A_TILE + B_TILE, &full[s], kx,
                                b_row0 + n0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- MMA issuer ----
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        const int chunk = kb / CHUNK_KB, kin = kb % CHUNK_KB;
        const uint32_t acc = tmem + (uint32_t)(chunk & 1) * BN;
        if (kin == 0)  // the epilogue must have drained this accumulator
          mbar_wait(&acc_empty[chunk & 1], ((chunk >> 1) & 1) ^ 1);
        mbar_wait(&full[s], ph);
        if (kb == 0)
          SGEMM_PHASE(2);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
        const uint32_t ah = base, al = base + A_TILE;
        const uint32_t bh = base + 2 * A_TILE, bl = bh + B_TILE;
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const uint32_t off = k * 32;  // 8 tf32 = 32 bytes along K
          const uint32_t acc0 = (kin | k) != 0;
          // B: 8 more K along a K-major row, or 8 more 128-byte rows (MN-major)
          const uint64_t dbh = BMN ? umma_desc_mn_sw128b32(bh + k * 1024) : umma_desc_sw64(bh + off);
          const uint64_t dbl = BMN ? umma_desc_mn_sw128b32(bl + k * 1024) : umma_desc_sw64(bl + off);
          mma_tf32<G::IDESC>(acc, umma_desc_sw64(al + off), dbh, acc0);  // small terms first
          mma_tf32<G::IDESC>(acc, umma_desc_sw64(ah + off), dbl, 1);
          mma_tf32<G::IDESC>(acc, umma_desc_sw64(ah + off), dbh, 1);
        }
        umma_commit(&empty[s]);  // the stage is free once these MMAs retire
        if (kin == CHUNK_KB - 1 || kb == nk - 1)
          umma_commit(&acc_full[chunk & 1]);
      }
      SGEMM_PHASE(3);
    }
    __syncwarp();
  } else {
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
    if (warp == 2 && lane == 0)
      SGEMM_PHASE(4);
    if (splits == 1) {
      // through the idle stage buffers (swizzled float4 granules, conflict
      // free both ways) so each warp stores whole rows: a thread's own row
      // would take one 16-byte segment per lane and instruction
      float4* part = reinterpret_cast<float4*>(smem);
#pragma unroll
      for (int j = 0; j < G::COLS; j += 4)
        part[partial_index<BN>(row, half * (G::COLS / 4) + j / 4)] =
            make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]);
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
      for (int r = warp - 2; r < BM; r += EPI_WARPS) {
        float* crow = C + (size_t)(m0 + r) * ldc + n0;
#pragma unroll
        for (int c4 = lane; c4 < BN / 4; c4 += 32)
          *reinterpret_cast<float4*>(crow + c4 * 4) = part[partial_index<BN>(r, c4)];
      }
    } else if (ws == nullptr || row / (BM / splits) == kz) {
      // partial tile into the (now idle) stage buffers: the last acc_full
      // commit follows every MMA, so no TMA write or MMA read is pending.
      // (With a workspace only the rows this CTA reduces stay here.)
      float4* part = reinterpret_cast<float4*>(smem);
#pragma unroll
      for (int j = 0; j < G::COLS; j += 4)
        part[partial_index<BN>(row, half * (G::COLS / 4) + j / 4)] =
            make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]);
    } else {
      // rows another CTA of the cluster reduces: to its workspace slice,
      // granule-major (lanes = consecutive rows = consecutive 16 bytes)
      const int rows = BM / splits, owner = row / rows;
      float4* slice = reinterpret_cast<float4*>(ws) +
                      (((size_t)bid * splits + owner) * splits + kz) * (size_t)(rows * BN / 4);
#pragma unroll
      for (int j = 0; j < G::COLS; j += 4)
        __stcg(slice + (size_t)(half * (G::COLS / 4) + j / 4) * rows + (row - owner * rows),
               make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0)
    SGEMM_PHASE(5);
  if (splits > 1 && ws != nullptr) {
    // split-K through L2: every CTA's slices for the peers went to the
    // workspace; after the cluster barrier (release / acquire: the peers'
    // global stores are visible) each CTA sums its rows in fixed z order
    cluster_sync();
    if (threadIdx.x == 0)
      SGEMM_PHASE(6);
    float* crow = C + (size_t)m0 * ldc + n0;
    switch (splits) {
      case 2: reduce_ws<BN, 2>(ws, smem, bid, kz, crow, ldc); break;
      case 4: reduce_ws<BN, 4>(ws, smem, bid, kz, crow, ldc); break;
      default: reduce_ws<BN, 8>(ws, smem, bid, kz, crow, ldc); break;
    }
  } else if (splits > 1) {
    cluster_sync();  // every partial of the cluster is written
    if (threadIdx.x == 0)
      SGEMM_PHASE(6);
    const int rows = BM / splits;
    // every peer's window once; the loads of all peers (and of two granules)
    // are issued before the first add, so the distributed-shared-memory
    // latency is paid once per pair of granules rather than once per peer
    uint32_t peer[kMaxSplits];
#pragma unroll
    for (int z = 0; z < kMaxSplits; ++z)
      peer[z] = z < splits ? cluster_map(smem_u32(smem), (uint32_t)z) : 0u;
    const int n4 = rows * (BN / 4);
    for (int i = threadIdx.x; i < n4; i += 2 * TC_THREADS) {
      const int i2 = i + TC_THREADS;
      const bool two = i2 < n4;
      const int r0 = kz * rows + i / (BN / 4), c0 = i % (BN / 4);
      const int r1 = kz * rows + i2 / (BN / 4), c1 = i2 % (BN / 4);
      const uint32_t off0 = (uint32_t)partial_index<BN>(r0, c0) * 16u;
      const uint32_t off1 = two ? (uint32_t)partial_index<BN>(r1, c1) * 16u : off0;
      float4 v0[kMaxSplits], v1[kMaxSplits];
#pragma unroll
      for (int z = 0; z < kMaxSplits; ++z)
        if (z < splits && z != kz) {
          v0[z] = ld_dsmem_f4(peer[z] + off0);
          v1[z] = ld_dsmem_f4(peer[z] + off1);
        }
      // this CTA's own partial through the local shared-memory path
      const float4 l0 = *reinterpret_cast<const float4*>(smem + off0);
      const float4 l1 = *reinterpret_cast<const float4*>(smem + off1);
      float4 a0 = kz == 0 ? l0 : v0[0], a1 = kz == 0 ? l1 : v1[0];
#pragma unroll
      for (int z = 1; z < kMaxSplits; ++z)
        if (z < splits) {
          const float4 w0 = z == kz ? l0 : v0[z], w1 = z == kz ? l1 : v1[z];
          a0.x = __fadd_rn(a0.x, w0.x);
          a0.y = __fadd_rn(a0.y, w0.y);
          a0.z = __fadd_rn(a0.z, w0.z);
          a0.w = __fadd_rn(a0.w, w0.w);
          a1.x = __fadd_rn(a1.x, w1.x);
          a1.y = __fadd_rn(a1.y, w1.y);
          a1.z = __fadd_rn(a1.z, w1.z);
          a1.w = __fadd_rn(a1.w, w1.w);
        }
      *reinterpret_cast<float4*>(C + (size_t)(m0 + r0) * ldc + n0 + c0 * 4) = a0;
      if (two)
        *reinterpret_cast<float4*>(C + (size_t)(m0 + r1) * ldc + n0 + c1 * 4) = a1;
    }
    cluster_sync();  // the peers are done reading this CTA's partial
  }
  if (threadIdx.x == 0)
    SGEMM_PHASE(7);
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(G::TMEM_COLS));
}

template <int BN, bool BMN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    sgemm_3xtf32_kernel(const __grid_constant__ CUtensorMap mAh,
                        const __grid_constant__ CUtensorMap mAl,
                        const __grid_constant__ CUtensorMap mBh,
                        const __grid_constant__ CUtensorMap mBl, float* __restrict__ C,
                        int M, int N, int K, int ldc, int splits, int a_row0,
                        int b_row0, int group_m, float* __restrict__ ws) {
  gemm_body<BN, BMN>(mAh, mAl, OneB{&mBh, &mBl}, C, M, N, K, ldc, splits, a_row0, b_row0,
                     group_m, ws);
}

// The multi-device fused path: this device's rows of A (raw + lo) times B
// whose K slices live on the context's devices (PeerB).
template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    sgemm_3xtf32_peer_kernel(const __grid_constant__ CUtensorMap mAh,
                             const __grid_constant__ CUtensorMap mAl,
                             const __grid_constant__ PeerB pb, float* __restrict__ C, int M,
                             int N, int K, int ldc, int group_m) {
  gemm_body<BN, true>(mAh, mAl, PeerBLoad{&pb}, C, M, N, K, ldc, 1, 0, 0, group_m, nullptr);
}

// ---- the 2-SM (CTA pair) GEMM kernel ------------------------------------------
// For C grids too small to fill the GPU (cfg2: 1024^3). A pair of CTAs on
// the two SMs of a TPC computes a 256 x BNP tile with tcgen05.mma
// .cta_group::2 (M = 256): each CTA loads its 128 rows of A and its BNP / 2
// columns of B, the leader's single thread issues the MMAs over both CTAs'
// shared memory, and each CTA's TMEM holds its 128 x BNP accumulator. Per SM
// this reads half as much B from shared memory as a 1-SM 128 x BNP tile, so
// a 256 x 128 pair tile runs the tensor core at the 1-SM 128 x 256 rate with
// half the accumulator: twice the tiles, half the split-K factor, and a
// third of the partial-tile bytes to exchange (the exchange bounds the small
// grids). Split-K pairs form a cluster of 2 x splits CTAs: rank = 2 z + q
// (z the K split, q the pair rank; rank 2 z is the pair's leader).
//
// Synchronisation: full[s] lives in the leader only; both CTAs' TMA loads
// (.cta_group::2) signal it, the leader arms it with both CTAs' bytes.
// empty[s] and acc_full[b] live in both CTAs; the leader's tcgen05.commit
// multicasts to the pair. acc_empty[b] lives in the leader and counts both
// CTAs' epilogue warps (remote arrives).
template <int BNP, bool BMN>
struct PairCfg {
  static constexpr int BH = BNP / 2;                           // B columns per CTA
  static constexpr int B_TILE = BH * BK * 4;                   // 4 / 8 KiB
  static constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;  // 24 / 32 KiB
  static constexpr int PSTAGES = BNP == 256 ? 6 : 8;
  static constexpr int SMEM_BYTES = PSTAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t TMEM_COLS = 2 * BNP;               // two accumulators
  static constexpr int COLS = BNP / 2;                         // epilogue: half a row
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    ((BMN ? 1u : 0u) << 16) |
                                    ((uint32_t)(BNP >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  static_assert(BM * BNP * 4 <= PSTAGES * STAGE_BYTES, "split-K partial must fit the stages");
  static_assert(!BMN || BH % 32 == 0, "MN-major B halves are 32-column chunks");
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map,
                                                 uint32_t bar_cluster, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map,
                                                 uint32_t bar_cluster, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y), "r"(z)
      : "memory");
}

template <uint32_t IDESC>
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t da, uint64_t db,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
               : "memory");
}

template <int BNP, bool BMN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    sgemm_3xtf32_pair_kernel(const __grid_constant__ CUtensorMap mAh,
                             const __grid_constant__ CUtensorMap mAl,
                             const __grid_constant__ CUtensorMap mBh,
                             const __grid_constant__ CUtensorMap mBl, float* __restrict__ C,
                             int M, int N, int K, int ldc, int splits, int a_row0, int b_row0,
                             int group_m, float* __restrict__ ws) {
  using G = PairCfg<BNP, BMN>;
  constexpr int STAGE_BYTES = G::STAGE_BYTES, B_TILE = G::B_TILE, BH = G::BH;
  constexpr int PSTAGES = G::PSTAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + PSTAGES * STAGE_BYTES);
  uint64_t* empty = full + PSTAGES;
  uint64_t* acc_full = empty + PSTAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0)
    SGEMM_PHASE(0);
  const uint32_t rank = cluster_rank();
  const int q = (int)(rank & 1), kz = (int)(rank >> 1);
  const uint32_t leader = rank & ~1u;
  const uint16_t pair_mask = (uint16_t)(3u << leader);

  // grouped raster over 256 x BNP pair tiles
  const int tiles_m = M / 256, tiles_n = N / BNP;
  const int per_group = group_m * tiles_n;
  const int bid = blockIdx.x / (2 * splits);  // pair tile (cluster) index
  const int first_m = (bid / per_group) * group_m;
  const int gsize = min(group_m, tiles_m - first_m);
  const int in_group = bid % per_group;
  const int m0 = (first_m + in_group % gsize) * 256 + q * BM;  // this CTA's rows
  const int n0 = (in_group / gsize) * BNP;                     // the pair tile's columns
  const int nb0 = n0 + q * BH;                                 // this CTA's B columns
  const int ksplit = K / splits;
  const int k_base = kz * ksplit;
  const int nk = ksplit / BK;
  CAFXG_DCHECK(bid < tiles_m * tiles_n && m0 + BM <= M && n0 + BNP <= N && nk > 0 &&
               ksplit % BK == 0);

  if (warp == 0 && lane == 0) {
    for (const CUtensorMap* m : {&mAh, &mAl, &mBh, &mBl})
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m))
                   : "memory");
    for (int s = 0; s < PSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2 * EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // both CTAs of the pair allocate together
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(G::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();  // the peers' barriers are initialised before any remote use
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0)
    SGEMM_PHASE(1);

  if (warp == 0) {
    // ---- TMA producer (both CTAs): this CTA's halves into its own stage,
    // completion counted on the leader's full[s]
    if (lane == 0) {
      const uint32_t full_leader = cluster_map(smem_u32(full), leader);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % PSTAGES;
        const uint32_t ph = (kb / PSTAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * STAGE_BYTES;
        const uint32_t fb = full_leader + 8u * s;
        if (q == 0)
          mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
        const int kx = k_base + kb * BK;
        tma_load_2d_pair(st, &mAh, fb, kx, a_row0 + m0);
        tma_load_2d_pair(st + A_TILE, &mAl, fb, kx, a_row0 + m0);
        if constexpr (BMN) {
          tma_load_3d_pair(st + 2 * A_TILE, &mBh, fb, 0, kx, (b_row0 + nb0) / 32);
          tma_load_3d_pair(st + 2 * A_TILE + B_TILE, &mBl, fb, 0, kx, (b_row0 + nb0) / 32);
        } else {
          tma_load_2d_pair(st + 2 * A_TILE, &mBh, fb, kx, b_row0 + nb0);
          tma_load_2d_pair(st + 2 * A_TILE + B_TILE, &mBl, fb, kx, b_row0 + nb0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- MMA issuer: the leader's lane 0 drives the pair ----
    if (lane == 0 && q == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % PSTAGES;
        const uint32_t ph = (kb / PSTAGES) & 1;
        const int chunk = kb / CHUNK_KB, kin = kb % CHUNK_KB;
        const uint32_t acc = tmem + (uint32_t)(chunk & 1) * BNP;
        if (kin == 0)  // both CTAs' epilogues must have drained this accumulator
          mbar_wait(&acc_empty[chunk & 1], ((chunk >> 1) & 1) ^ 1);
        mbar_wait(&full[s], ph);
        if (kb == 0)
          SGEMM_PHASE(2);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
        const uint32_t ah = base, al = base + A_TILE;
        const uint32_t bh = base + 2 * A_TILE, bl = bh + B_TILE;
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const uint32_t off = k * 32;
          const uint32_t acc0 = (kin | k) != 0;
          const uint64_t dbh = BMN ? umma_desc_mn_sw128b32(bh + k * 1024) : umma_desc_sw64(bh + off);
          const uint64_t dbl = BMN ? umma_desc_mn_sw128b32(bl + k * 1024) : umma_desc_sw64(bl + off);
          mma_tf32_pair<G::IDESC>(acc, umma_desc_sw64(al + off), dbh, acc0);
          mma_tf32_pair<G::IDESC>(acc, umma_desc_sw64(ah + off), dbl, 1);
          mma_tf32_pair<G::IDESC>(acc, umma_desc_sw64(ah + off), dbh, 1);
        }
        umma_commit_pair(&empty[s], pair_mask);  // both CTAs' stage s is free
        if (kin == CHUNK_KB - 1 || kb == nk - 1)
          umma_commit_pair(&acc_full[chunk & 1], pair_mask);
      }
      SGEMM_PHASE(3);
    }
    __syncwarp();
  } else {
    // ---- epilogue (both CTAs): this CTA's 128 rows from its own TMEM ----
    const int q4 = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = q4 * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const uint32_t acc_empty_leader = cluster_map(smem_u32(acc_empty), leader);
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
        tmem_ld32(tmem + lane_base + (uint32_t)(b * BNP + half * G::COLS + c * 32), r);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          sum[c * 32 + j] = __fadd_rn(sum[c * 32 + j], __uint_as_float(r[j]));
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        mbar_arrive_cluster(acc_empty_leader + 8u * b);
    }
    if (warp == 2 && lane == 0)
      SGEMM_PHASE(4);
    if (splits == 1) {
      // through the idle stage buffers (swizzled float4 granules, conflict
      // free both ways) so each warp stores whole rows: a thread's own row
      // would take one 16-byte segment per lane and instruction
      float4* part = reinterpret_cast<float4*>(smem);
#pragma unroll
      for (int j = 0; j < G::COLS; j += 4)
        part[partial_index<BNP>(row, half * (G::COLS / 4) + j / 4)] =
            make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]);
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_WARPS * 32) : "memory");
      for (int r = warp - 2; r < BM; r += EPI_WARPS) {
        float* crow = C + (size_t)(m0 + r) * ldc + n0;
#pragma unroll
        for (int c4 = lane; c4 < BNP / 4; c4 += 32)
          *reinterpret_cast<float4*>(crow + c4 * 4) = part[partial_index<BNP>(r, c4)];
      }
    } else if (row / (BM / splits) == kz) {
      float4* part = reinterpret_cast<float4*>(smem);
#pragma unroll
      for (int j = 0; j < G::COLS; j += 4)
        part[partial_index<BNP>(row, half * (G::COLS / 4) + j / 4)] =
            make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]);
    } else {
      // rows the same-q CTA of split `owner` reduces: to the workspace; the
      // 128-row half tiles (pair tile * 2 + q) index it like 1-SM tiles
      const int rows = BM / splits, owner = row / rows;
      const int htile = bid * 2 + q;
      float4* slice = reinterpret_cast<float4*>(ws) +
                      (((size_t)htile * splits + owner) * splits + kz) * (size_t)(rows * BNP / 4);
#pragma unroll
      for (int j = 0; j < G::COLS; j += 4)
        __stcg(slice + (size_t)(half * (G::COLS / 4) + j / 4) * rows + (row - owner * rows),
               make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0)
    SGEMM_PHASE(5);
  cluster_sync();  // partials visible; the pair's MMAs and TMEM reads are over
  if (threadIdx.x == 0)
    SGEMM_PHASE(6);
  if (splits > 1) {
    float* crow = C + (size_t)m0 * ldc + n0;
    const int htile = bid * 2 + q;
    switch (splits) {
      case 2: reduce_ws<BNP, 2>(ws, smem, htile, kz, crow, ldc); break;
      default: reduce_ws<BNP, 4>(ws, smem, htile, kz, crow, ldc); break;
    }
  }
  if (threadIdx.x == 0)
    SGEMM_PHASE(7);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
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
  SPLIT_SPAN_BEGIN();
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
    SPLIT_SPAN_END();
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
  SPLIT_SPAN_END();
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

// lo half for operands the GEMM reads raw: the tensor core takes a 32-bit
// operand as tf32 by dropping its low 13 mantissa bits, so the fp32 value
// itself is hi = trunc_tf32(x); lo = rna_tf32(x - hi) (the difference is
// exact in fp32). Dropped terms: lo(A)*lo(B) <= 2^-20 relative and lo's own
// rounding <= 2^-21, below the fp32 accumulation's error.
__device__ __forceinline__ float lo_tf32(float x) {
  const float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  uint32_t l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(__fsub_rn(x, hi)));
  return __uint_as_float(l);
}

__device__ __forceinline__ float4 lo_tf32(float4 v) {
  return make_float4(lo_tf32(v.x), lo_tf32(v.y), lo_tf32(v.z), lo_tf32(v.w));
}

// rows x cols (pitch ld_in, float4-aligned) -> lo halves packed (pitch cols);
// thread t of `nthreads` takes float4 granules t, t + nthreads, ... four at
// a time (four loads in flight before the first store)
__device__ __forceinline__ void lo_rows(const float* __restrict__ in, int ld_in, int rows,
                                        int cols, float* __restrict__ out, uint32_t t,
                                        uint32_t nthreads) {
  const uint32_t c4 = (uint32_t)cols / 4, total = (uint32_t)rows * c4;
  for (uint32_t i = t; i < total; i += 4 * nthreads) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t j = i + u * nthreads;
      if (j < total) {
        const uint32_t r = j / c4, c = (j - r * c4) * 4;
        v[u] = __ldcs(reinterpret_cast<const float4*>(in + (size_t)r * ld_in + c));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t j = i + u * nthreads;
      if (j < total)
        *reinterpret_cast<float4*>(out + (size_t)j * 4) = lo_tf32(v[u]);
    }
  }
}

// One launch for both operands: blocks [0, nb_a) make lo(A) (M x K), the
// rest lo(B) (K x N, B's own layout). The grid is at most 4 CTAs of 256
// threads per SM, so the dependent GEMM's CTAs (320 threads) fit beside it:
// the trigger comes first, the GEMM's prologue (barriers, TMEM, tensor-map
// prefetch) overlaps this pass and its griddepcontrol.wait still waits for
// the whole grid.
__global__ void __launch_bounds__(256) split_lo_kernel(const float* __restrict__ A, int lda,
                                                       int M, int K, float* __restrict__ Al,
                                                       const float* __restrict__ B, int ldb,
                                                       int N, float* __restrict__ Bl,
                                                       int nb_a) {
  asm volatile("griddepcontrol.launch_dependents;");
  SPLIT_SPAN_BEGIN();
  if ((int)blockIdx.x < nb_a)
    lo_rows(A, lda, M, K, Al, blockIdx.x * blockDim.x + threadIdx.x, (uint32_t)nb_a * blockDim.x);
  else
    lo_rows(B, ldb, K, N, Bl, (blockIdx.x - nb_a) * blockDim.x + threadIdx.x,
            (gridDim.x - (uint32_t)nb_a) * blockDim.x);
  SPLIT_SPAN_END();
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

// rows x cols fp32 row-major with row pitch `ld` floats; box = box_cols
// (contiguous) x box_rows
bool make_map(CUtensorMap* m, const float* base, int rows, int cols, int ld, int box_cols,
              int box_rows, CUtensorMapSwizzle swz) {
  EncodeTiled enc = get_encoder();
  if (!enc)
    return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K-major operand (rows of K): BK x box_rows boxes, SWIZZLE_64B
bool make_map_kmajor(CUtensorMap* m, const float* base, int rows, int K, int ld, int box_rows) {
  return make_map(m, base, rows, K, ld, BK, box_rows, CU_TENSOR_MAP_SWIZZLE_64B);
}

// MN-major B (K rows of N) as a 3-D tensor (32 columns, K rows, N / 32
// column chunks): one box of 32 x BK x bn / 32 fills a stage's B tile in
// the chunked SWIZZLE_128B_ATOM_32B layout with one TMA request
bool make_map_mnmajor(CUtensorMap* m, const float* base, int K, int N, int ld, int bn) {
  EncodeTiled enc = get_encoder();
  if (!enc || N % 32)
    return false;
  cuuint64_t dims[3] = {32, (cuuint64_t)K, (cuuint64_t)N / 32};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 4, 128};
  cuuint32_t box[3] = {32, (cuuint32_t)BK, (cuuint32_t)bn / 32};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool sgemm_tc_supported(int M, int N, int K, int lda, int ldb, int ldc) {
  (void)ldb;
  return M >= BM && N >= 128 && K >= BK && M % BM == 0 && N % 128 == 0 && K % 32 == 0 &&
         lda % 4 == 0 && ldc % 4 == 0 && get_encoder() != nullptr;
}

size_t sgemm_tc_ws_bytes(int M, int N, int splits, int bn) {
  // per cluster (one C tile): for every reducing CTA one slice of BM / splits
  // rows per source CTA (its own slot unused), i.e. `splits` partial tiles
  if (splits <= 1)
    return 0;
  return (size_t)(M / BM) * (N / bn) * splits * BM * bn * sizeof(float);
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

template <int BN, bool BMN>
void configure_once() {
  // once per device (the attribute is per-device state)
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !(configured.load() >> dev & 1)) {
    cudaFuncSetAttribute(sgemm_3xtf32_kernel<BN, BMN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN, BMN>::SMEM_BYTES);
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
  configure_once<BN, false>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(splits * 256));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = Cfg<BN, false>::SMEM_BYTES;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, sgemm_3xtf32_kernel<BN, false>, &cfg) != cudaSuccess ||
      n < 1) {
    cudaGetLastError();
    n = 148 / splits;
  }
  cache[splits].store(n);
  return n;
}

// Raw operands: the GEMM reads A and B through TMA as they lie (both
// 16-byte aligned with 16-byte row pitches) and only their lo halves are
// materialised -- half the split pass's writes and no transpose -- but the
// MN-major B operand costs ~5% of MMA throughput (2048^3: 64 against 61 us
// of MMA). Taken where the split pass weighs more than that: the pass
// scales with M + N, the GEMM with M * N, and M N / (M + N) < 3200 covers up
// to ~6400^2 (measured: 4096^3 0.622 -> 0.590 ms, 16384^3 38.4 -> 40.4 ms).
// CAFXG_SGEMM_RAW=0 / 1 forces either way (experiments).
bool use_raw_operands(const float* A, int lda, const float* B, int ldb, int M, int N) {
  static const int env = [] {
    const char* e = getenv("CAFXG_SGEMM_RAW");
    return e ? atoi(e) : -1;
  }();
  if (((uintptr_t)A & 15) || ((uintptr_t)B & 15) || lda % 4 || ldb % 4 || env == 0)
    return false;
  return env == 1 || (double)M * N / ((double)M + N) < 3200.0;
}

// CAFXG_SGEMM_WS=0: split-K reduces through distributed shared memory even
// where a workspace is available (experiments)
bool ws_enabled() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_SGEMM_WS");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CAFXG_SGEMM_PDL=0 launches the GEMM without programmatic dependent launch
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("CAFXG_SGEMM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int BN, bool BMN>
int launch(const CUtensorMap* m, float* C, int M, int N, int K, int ldc, void* stream,
           int splits, int a_row0, int b_row0, float* ws) {
  configure_once<BN, BMN>();
  if (splits < 1 || splits > kMaxSplits || (splits & (splits - 1)) ||
      K % (16 * splits) != 0)
    splits = 1;
  const int tiles = (M / BM) * (N / BN);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(tiles * splits));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = Cfg<BN, BMN>::SMEM_BYTES;
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
  cudaLaunchKernelEx(&cfg, sgemm_3xtf32_kernel<BN, BMN>, m[0], m[1], m[2], m[3], C, M, N, K, ldc,
                     splits, a_row0, b_row0, group_m, splits > 1 ? ws : nullptr);
  return (int)cudaGetLastError();
}

// ---- CTA-pair kernel (256 x 128 pair tiles) ----

constexpr int kMaxPairSplits = 4;  // cluster of 2 x 4 CTAs: the portable maximum

// pair tile width (columns): CAFXG_SGEMM_PAIR_BN=128 / 256 (experiments)
int pair_bn() {
  static const int v = [] {
    const char* e = getenv("CAFXG_SGEMM_PAIR_BN");
    return e && atoi(e) == 128 ? 128 : 256;
  }();
  return v;
}

template <int BNP, bool BMN>
void configure_pair_once() {
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !(configured.load() >> dev & 1)) {
    cudaFuncSetAttribute(sgemm_3xtf32_pair_kernel<BNP, BMN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PairCfg<BNP, BMN>::SMEM_BYTES);
    configured.fetch_or(1ull << dev);
  }
}

template <int BNP>
int max_active_pair_clusters(int splits) {
  static std::atomic<int> cache[kMaxPairSplits + 1];
  int v = cache[splits].load();
  if (v)
    return v;
  configure_pair_once<BNP, false>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * splits * 128));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = PairCfg<BNP, false>::SMEM_BYTES;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)(2 * splits);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, sgemm_3xtf32_pair_kernel<BNP, false>, &cfg) !=
          cudaSuccess ||
      n < 1) {
    cudaGetLastError();
    n = 148 / (2 * splits);
  }
  cache[splits].store(n);
  return n;
}

// CAFXG_SGEMM_PAIR=0 never takes the CTA-pair kernel, =1 takes it for every
// eligible shape (experiments); default: grids that fill the GPU without
// split-K (measured, b2b: 2048^3 79.8 -> 78.5 us, 4096^3 0.585 -> 0.568 ms,
// 16384^3 41.0 -> 39.9 ms; at 1024^3, where the 1-SM grid splits K 4 ways,
// the pair kernel's 256 x 256 tiles need the same 4-way exchange and its
// 8-CTA clusters fit fewer at once: 31 against 23 us)
bool pair_allowed(int force) {
  static const int env = [] {
    const char* e = getenv("CAFXG_SGEMM_PAIR");
    return e ? atoi(e) : -1;
  }();
  return force ? env == 1 : env != 0;
}

int pair_splits(int M, int N, int K, int bnp) {
  const int tiles = (M / 256) * (N / bnp);
  int s = 1;
  while (s < kMaxPairSplits && K % (16 * s * 2) == 0 && K / (s * 2) >= 128 &&
         tiles <= (bnp == 256 ? max_active_pair_clusters<256>(s * 2)
                              : max_active_pair_clusters<128>(s * 2)))
    s *= 2;
  return s;
}

template <int BNP, bool BMN>
int launch_pair(const CUtensorMap* m, float* C, int M, int N, int K, int ldc, void* stream,
                int splits, int a_row0, int b_row0, float* ws) {
  configure_pair_once<BNP, BMN>();
  if (splits < 1 || splits > kMaxPairSplits || (splits & (splits - 1)) ||
      K % (16 * splits) != 0 || ws == nullptr)
    splits = 1;  // split-K pairs reduce through the workspace only
  const int tiles = (M / 256) * (N / BNP);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(tiles * 2 * splits));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = PairCfg<BNP, BMN>::SMEM_BYTES;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)(2 * splits);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  // raster groups of 4 pair tiles (1024 A rows). At 16384^3 (ncu, DRAM read
  // per GEMM; CUDA events back to back): 16 pair tiles 84 GB, 40.1 ms; 8:
  // 57 GB, 38.1 ms; 4: 54 GB, 37.4 ms; 2: 38.9 ms
  static const int group_m = [] {
    const char* e = getenv("CAFXG_SGEMM_GROUP_M");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : 4;
  }();
  cudaLaunchKernelEx(&cfg, sgemm_3xtf32_pair_kernel<BNP, BMN>, m[0], m[1], m[2], m[3], C, M,
                     N, K, ldc, splits, a_row0, b_row0, group_m, ws);
  return (int)cudaGetLastError();
}

int launch_peer(const CUtensorMap* mA, const PeerB& pb, float* C, int M, int N, int K, int ldc,
                void* stream) {
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !(configured.load() >> dev & 1)) {
    cudaFuncSetAttribute(sgemm_3xtf32_peer_kernel<256>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<256, true>::SMEM_BYTES);
    configured.fetch_or(1ull << dev);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((M / BM) * (N / 256)));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = Cfg<256, true>::SMEM_BYTES;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, sgemm_3xtf32_peer_kernel<256>, mA[0], mA[1], pb, C, M, N, K, ldc,
                     GROUP_M);
  return (int)cudaGetLastError();
}

// Which kernel, tile width and split-K factor a device-API GEMM takes (the
// scratch size and the launch must agree): the CTA-pair kernel (256 x 256
// pair tiles) where the 1-SM grid needs no split-K, else 1-SM tiles.
struct TcPlan {
  bool pair;
  int bn;
  int splits;
};

TcPlan tc_plan(int M, int N, int K, int sms, int splits_req) {
  TcPlan p{false, sgemm_tc_pick_bn(M, N, sms), 1};
  const int s1 = sgemm_tc_splits(M, N, K, sms, p.bn);
  const int bnp = pair_bn();
  const bool eligible = M % 256 == 0 && N % bnp == 0 && splits_req <= kMaxPairSplits;
  if (eligible && pair_allowed(0) && (s1 == 1 || pair_allowed(1))) {
    p.pair = true;
    p.bn = bnp;
    p.splits = splits_req > 0 ? splits_req : pair_splits(M, N, K, bnp);
    return p;
  }
  p.splits = splits_req > 0 ? splits_req : s1;
  return p;
}

}  // namespace

size_t sgemm_tc_scratch_bytes(int M, int N, int K, int sm_count, int splits_req) {
  // hi/lo splits of A and B^T (the raw-operand path uses the first half: lo
  // of A and B) and the split-K workspace
  const TcPlan p = tc_plan(M, N, K, sm_count > 0 ? sm_count : 148, splits_req);
  return ((size_t)M * K * 2 + (size_t)N * K * 2) * sizeof(float) +
         sgemm_tc_ws_bytes(M, N, p.splits, p.bn);
}

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
  maps->b_mn_major = false;
  maps->pair = false;
  if (!make_map_kmajor(&m[0], Ah, a_rows, K, K, BM) ||
      !make_map_kmajor(&m[1], Al, a_rows, K, K, BM) ||
      !make_map_kmajor(&m[2], Bh, N, K, K, bn) || !make_map_kmajor(&m[3], Bl, N, K, K, bn))
    return (int)cudaErrorInvalidValue;
  return 0;
}

int sgemm_tc_make_maps_raw(const float* A, int lda, const float* Al, int a_rows,
                           const float* B, int ldb, const float* Bl, int N, int K, int bn,
                           SgemmTcMaps* maps) {
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(maps->m);
  maps->bn = bn;
  maps->b_mn_major = true;
  maps->pair = false;
  if (!make_map_kmajor(&m[0], A, a_rows, K, lda, BM) ||
      !make_map_kmajor(&m[1], Al, a_rows, K, K, BM) || !make_map_mnmajor(&m[2], B, K, N, ldb, bn) ||
      !make_map_mnmajor(&m[3], Bl, K, N, N, bn))
    return (int)cudaErrorInvalidValue;
  return 0;
}

int sgemm_tc_gemm_maps(const SgemmTcMaps* maps, float* C, int M, int N, int K, int ldc,
                       void* stream, int splits, int a_row0, int b_row0, float* ws) {
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(maps->m);
  if (maps->pair) {  // maps->bn: each CTA's half of the pair tile's columns
    if (maps->bn == 128)
      return maps->b_mn_major
                 ? launch_pair<256, true>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0, ws)
                 : launch_pair<256, false>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0, ws);
    return maps->b_mn_major
               ? launch_pair<128, true>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0, ws)
               : launch_pair<128, false>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0, ws);
  }
  if (maps->b_mn_major)
    return maps->bn == 256
               ? launch<256, true>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0, ws)
               : launch<128, true>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0, ws);
  return maps->bn == 256
             ? launch<256, false>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0, ws)
             : launch<128, false>(m, C, M, N, K, ldc, stream, splits, a_row0, b_row0, ws);
}

bool sgemm_tc_raw_wanted(int M, int N) {
  // the size rule of use_raw_operands for buffers the runtime allocates
  // (16-byte aligned, packed)
  static const int env = [] {
    const char* e = getenv("CAFXG_SGEMM_RAW");
    return e ? atoi(e) : -1;
  }();
  if (env == 0)
    return false;
  return env == 1 || (double)M * N / ((double)M + N) < 3200.0;
}

bool sgemm_tc_pair_wanted(int M, int N, int K, int sms) {
  const TcPlan p = tc_plan(M, N, K, sms > 0 ? sms : 148, 0);
  return p.pair && p.splits == 1 && p.bn == 256;
}

int sgemm_tc_make_pair_maps(const float* Ah, const float* Al, int a_rows, const float* Bh,
                            const float* Bl, int N, int K, SgemmTcMaps* maps) {
  // each CTA of a pair loads 128 of the pair tile's 256 B^T rows
  if (int e = sgemm_tc_make_maps(Ah, Al, a_rows, Bh, Bl, N, K, 128, maps))
    return e;
  maps->pair = true;
  return 0;
}

int sgemm_tc_lo(const float* X, int ld, int rows, int cols, float* out, int sm_count,
                void* stream) {
  if (rows <= 0 || cols <= 0)
    return 0;
  if (((uintptr_t)X & 15) || ((uintptr_t)out & 15) || ld % 4 || cols % 4 ||
      (size_t)rows * cols / 4 >= (1ull << 32))
    return (int)cudaErrorInvalidValue;
  const int sms = sm_count > 0 ? sm_count : 148;
  const size_t g4 = (size_t)rows * cols / 4;
  const int grid = std::max(1, (int)std::min<size_t>((g4 + 1023) / 1024, (size_t)sms * 4));
  // every block takes the first operand; the second is empty
  split_lo_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(X, ld, rows, cols, out, nullptr, 0, 0,
                                                          nullptr, grid);
  return (int)cudaGetLastError();
}

bool sgemm_tc_peer_supported(int M, int N, int K, int nslices) {
  return nslices >= 1 && nslices <= kMaxPeerSlices && M % BM == 0 && N % 256 == 0 &&
         K % nslices == 0 && (K / nslices) % BK == 0 && get_encoder() != nullptr;
}

int sgemm_tc_peer_gemm(const float* A, int lda, const float* Alo, int M, int N, int K,
                       const float* const* Bs, const float* const* Blos, int nslices, float* C,
                       int ldc, void* stream) {
  if (!sgemm_tc_peer_supported(M, N, K, nslices) || lda % 4 || ldc % 4 ||
      ((uintptr_t)A & 15) || ((uintptr_t)C & 15))
    return (int)cudaErrorInvalidValue;
  if (M == 0)
    return 0;
  const int kslice = K / nslices;
  CUtensorMap mA[2];
  PeerB pb{};
  pb.kslice = kslice;
  pb.n = nslices;
  if (!make_map_kmajor(&mA[0], A, M, K, lda, BM) || !make_map_kmajor(&mA[1], Alo, M, K, K, BM))
    return (int)cudaErrorInvalidValue;
  for (int i = 0; i < nslices; ++i)
    if (!make_map_mnmajor(&pb.h[i], Bs[i], kslice, N, N, 256) ||
        !make_map_mnmajor(&pb.l[i], Blos[i], kslice, N, N, 256))
      return (int)cudaErrorInvalidValue;
  return launch_peer(mA, pb, C, M, N, K, ldc, stream);
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
  if ((size_t)M * K / 4 >= (1ull << 32))  // the A split indexes float4s in 32 bits
    return (int)cudaErrorInvalidValue;
  const int sms = sm_count > 0 ? sm_count : 148;
  const TcPlan plan = tc_plan(M, N, K, sms, splits_req);
  // the pair kernel's CTAs each load half of the pair tile's B columns
  const int bn = plan.pair ? plan.bn / 2 : plan.bn;
  const int splits = plan.splits;
  float* Ah = static_cast<float*>(scratch);
  float* Al = Ah + (size_t)M * K;
  float* Bh = Al + (size_t)M * K;
  float* Bl = Bh + (size_t)N * K;
  float* ws = Bl + (size_t)N * K;  // split-K workspace (sgemm_tc_scratch_bytes)
  // maps before the first launch: the two launches then go out back to back
  // (encoding between them left the GPU idle for the host's encode time)
  SgemmTcMaps maps;
  if (use_raw_operands(A, lda, B, ldb, M, N) && (size_t)K * N / 4 < (1ull << 32)) {
    // lo halves only, into the first half of the scratch; the GEMM reads A
    // and B themselves as the hi halves
    float* Alo = Ah;
    float* Blo = Alo + (size_t)M * K;
    if (int me = sgemm_tc_make_maps_raw(A, lda, Alo, M, B, ldb, Blo, N, K, bn, &maps))
      return me;
    const size_t ga = (size_t)M * K / 4, gb = (size_t)K * N / 4;
    const int grid = std::max<int>(2, (int)std::min<size_t>((ga + gb + 1023) / 1024,
                                                            (size_t)sms * 4));
    const int nb_a = std::clamp((int)((double)grid * ga / (ga + gb) + 0.5), 1, grid - 1);
    split_lo_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A, lda, M, K, Alo, B, ldb, N, Blo,
                                                            nb_a);
  } else {
    if (int me = sgemm_tc_make_maps(Ah, Al, M, Bh, Bl, N, K, bn, &maps))
      return me;
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
  }
  maps.pair = plan.pair;
  int e = (int)cudaGetLastError();
  if (e == 0)
    e = sgemm_tc_gemm_maps(&maps, C, M, N, K, ldc, stream, splits, 0, 0,
                           ws_enabled() || plan.pair ? ws : nullptr);
  if (launches)
    *launches = 2;
  return e;
}

}  // namespace cafxg

#ifdef CAFXG_SGEMM_PHASES
// tools/sgemm_phases.py: reset before a launch, read after it
extern "C" int cafxg_debug_sgemm_phases(unsigned long long* out, int nblocks,
                                        unsigned long long* split_span, int reset) {
  using namespace cafxg;
  if (reset) {
    static unsigned long long zero[1024][16];
    unsigned long long span0[2] = {~0ull, 0ull};
    cudaMemcpyToSymbol(g_sgemm_phase, zero, sizeof(zero));
    return (int)cudaMemcpyToSymbol(g_split_span, span0, sizeof(span0));
  }
  cudaMemcpyFromSymbol(out, g_sgemm_phase, (size_t)std::min(nblocks, 1024) * 16 * 8);
  return (int)cudaMemcpyFromSymbol(split_span, g_split_span, 16);
}
#endif
