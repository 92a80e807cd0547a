// fp32 GEMM launchers for the `matrix_multiply` compute actor.
#pragma once
#include <cstddef>
#include <cstdint>

namespace cafxg {

// Register-tiled FFMA kernel; any shape, any leading dims.
int sgemm_simt_launch(const float* A, const float* B, float* C, int M, int N,
                      int K, int lda, int ldb, int ldc, void* stream);

// 3xTF32 tcgen05 path (sgemm_tc.cu). Shape constraints are checked by
// sgemm_tc_supported (the caller also checks 16-byte alignment of A and C);
// scratch holds the tf32 hi/lo splits of A and B^T, or the lo halves of A and
// B for raw operands, and the split-K workspace (sgemm_tc_scratch_bytes).
// sgemm_tc_launch picks the kernel (1-SM tiles or CTA pairs), the operand form
// and the split-K factor per shape (tc_plan).
bool sgemm_tc_supported(int M, int N, int K, int lda, int ldb, int ldc);
size_t sgemm_tc_scratch_bytes(int M, int N, int K, int sm_count, int splits_req = 0);
// splits: split-K cluster size (1/2/4/8), 0 = the plan's choice
int sgemm_tc_launch(const float* A, const float* B, float* C, int M, int N,
                    int K, int lda, int ldb, int ldc, void* scratch,
                    int sm_count, void* stream, int* launches, int splits = 0);
// The three stages separately (pipelined host requests): tf32 hi/lo split of
// an A row block (M x K, packed out), split + transpose of B (to N x K), and
// the GEMM on split operands.
int sgemm_tc_split_a(const float* A, int lda, int M, int K, float* Ah, float* Al,
                     void* stream);
int sgemm_tc_split_b(const float* B, int ldb, int K, int N, float* Bh, float* Bl,
                     void* stream);
int sgemm_tc_gemm(const float* Ah, const float* Al, const float* Bh, const float* Bl,
                  float* C, int M, int N, int K, int ldc, void* stream, int splits = 1,
                  int bn = 256);
// The four TMA tensor maps of a GEMM (A_hi, A_lo over a_rows rows; B_hi,
// B_lo), encoded once and reused by launches over the same buffers: a row
// block of m <= a_rows rows only touches rows below m.
struct SgemmTcMaps {
  alignas(64) unsigned char m[4][128];
  int bn;           // tile width the maps were encoded for (B box rows)
  bool b_mn_major;  // B operands as they lie (K x N) rather than B^T (N x K)
  bool pair;        // CTA-pair kernel (bn = its per-CTA half of the pair tile's columns)
};
int sgemm_tc_make_maps(const float* Ah, const float* Al, int a_rows, const float* Bh,
                       const float* Bl, int N, int K, int bn, SgemmTcMaps* maps);
// The same for raw operands: A (pitch lda) and B (K x N, pitch ldb) are read
// as their own hi halves (the tensor core truncates fp32 to tf32); Al (pitch
// K) and Bl (K x N, pitch N) hold the lo halves. b_row0 of a launch is then
// B's first column.
int sgemm_tc_make_maps_raw(const float* A, int lda, const float* Al, int a_rows,
                           const float* B, int ldb, const float* Bl, int N, int K, int bn,
                           SgemmTcMaps* maps);
// a_row0 / b_row0: this GEMM's first row inside the mapped A / B^T (block
// (i, j) of a larger product whose maps were encoded once)
// ws: split-K workspace (sgemm_tc_ws_bytes) for a reduction through L2;
// null reduces through distributed shared memory
int sgemm_tc_gemm_maps(const SgemmTcMaps* maps, float* C, int M, int N, int K, int ldc,
                       void* stream, int splits, int a_row0 = 0, int b_row0 = 0,
                       float* ws = nullptr);
size_t sgemm_tc_ws_bytes(int M, int N, int splits, int bn);
// lo halves of one operand (rows x cols, pitch ld) for the raw-operand GEMMs:
// lo = rna_tf32(x - trunc_tf32(x)), packed (pitch cols)
int sgemm_tc_lo(const float* X, int ld, int rows, int cols, float* out, int sm_count,
                void* stream);
// The multi-device fused GEMM: C (M x N) = A (M x K, raw + lo) times B whose
// K slices (K / nslices rows of N floats each, raw + lo, pitch N) live in the
// memory of the context's devices -- the kernel's TMA loads pull each k-block
// from the slice's device over NVLink (peer access enabled), so B is never
// gathered. M % 128 == 0, N % 256 == 0, K / nslices a multiple of 16.
bool sgemm_tc_peer_supported(int M, int N, int K, int nslices);
int sgemm_tc_peer_gemm(const float* A, int lda, const float* Alo, int M, int N, int K,
                       const float* const* Bs, const float* const* Blos, int nslices, float* C,
                       int ldc, void* stream);
// CTA-pair kernel (256 x 256 pair tiles, tcgen05 .cta_group::2) for split
// operands: whether an M x N x K product should take it (a grid that needs no
// split-K), and its maps (launched by sgemm_tc_gemm_maps with splits 1; blocks
// of it need M % 256 == N % 256 == 0)
bool sgemm_tc_pair_wanted(int M, int N, int K, int sms);
// whether an M x N product should take the raw-operand form (lo-only pass,
// MN-major B): the device-API size rule, for the runtime's own buffers
bool sgemm_tc_raw_wanted(int M, int N);
int sgemm_tc_make_pair_maps(const float* Ah, const float* Al, int a_rows, const float* Bh,
                            const float* Bl, int N, int K, SgemmTcMaps* maps);
// tile width (256 or 128 columns) and split-K factor (thread-block cluster
// size, <= 8) for a C grid
int sgemm_tc_pick_bn(int M, int N, int sms);
int sgemm_tc_splits(int M, int N, int K, int sms, int bn);

// Device FNV-1a-64 over u32 cells hashed big-endian (fnv.cu).
size_t fnv_scratch_bytes(uint64_t n, int sms);
int fnv_launch(const uint32_t* cells, uint64_t n, uint64_t seed, uint64_t* out,
               void* scratch, int sms, void* stream, int* launches);
// The same in two parts, so the seed-independent pass 1 (per-segment
// low-byte tables, the bulk of the work) can run on segments as soon as
// their cells exist: segments are fnv_segments() cells long.
void fnv_segments(uint64_t n, int sms, uint64_t* seg_cells, uint32_t* nseg);
int fnv_lowbyte_launch(const uint32_t* cells, uint64_t n, uint32_t seg_begin,
                       uint32_t seg_count, void* scratch, int sms, void* stream);
int fnv_finish_launch(const uint32_t* cells, uint64_t n, uint64_t seed, uint64_t* out,
                      void* scratch, int sms, void* stream, int* launches);

}  // namespace cafxg
