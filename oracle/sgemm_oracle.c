/*
 * TEST INFRASTRUCTURE ONLY -- CPU checker and builder-authored CPU baseline for
 * the fp32 matrix_multiply compute actor.
 *
 * The reference has no matmul implementation: the kernel exists only as the
 * OpenCL prototype `matrix_multiply(float* matrix1, float* matrix2, float*
 * output)` behind
 * `spawn_cl<float*(float*,float*)>(source, "matrix_multiply", {size, size})`
 * (PAPER.md:357-361): 1-D row-major arrays, last parameter is the output.
 * Parity is therefore pinned only by the BASELINE.json check: sampled rows
 * against an fp64-accumulated sum_k (double)A_ik * (double)B_kj, normwise
 * max_j |dC_ij| / max_j |R_ij| <= 1e-5.
 *
 * Inputs come from a counter-based seeded generator (splitmix64 of
 * seed + index), so host and device can produce identical operands and a
 * test can regenerate any element without storing the matrix.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* uniform[-1,1) with 24 random bits: k * 2^-23 - 1, k in [0, 2^24). Exact in
 * binary32. Must match paper_1505_07368_b200/csrc/sgemm_common.cuh. */
static inline float uniform_pm1(uint64_t seed, uint64_t idx) {
  uint64_t r = splitmix64(seed * 0xd1342543de82ef95ull + idx);
  int32_t k = (int32_t)(r >> 40);
  return (float)k * (1.0f / 8388608.0f) - 1.0f;
}

typedef struct {
  float* dst;
  size_t begin, end;
  uint64_t seed, offset;
} fill_job;

static void* fill_worker(void* arg) {
  fill_job* j = (fill_job*)arg;
  for (size_t i = j->begin; i < j->end; ++i)
    j->dst[i] = uniform_pm1(j->seed, j->offset + i);
  return NULL;
}

void oracle_fill_uniform(float* dst, size_t n, uint64_t seed, uint64_t offset,
                         uint32_t threads) {
  if (threads == 0)
    threads = 1;
  pthread_t* tids = (pthread_t*)calloc(threads, sizeof(pthread_t));
  fill_job* jobs = (fill_job*)calloc(threads, sizeof(fill_job));
  size_t per = (n + threads - 1) / threads;
  for (uint32_t k = 0; k < threads; ++k) {
    size_t b = (size_t)k * per, e = b + per;
    if (b > n) b = n;
    if (e > n) e = n;
    jobs[k] = (fill_job){dst, b, e, seed, offset};
    pthread_create(&tids[k], NULL, fill_worker, &jobs[k]);
  }
  for (uint32_t k = 0; k < threads; ++k)
    pthread_join(tids[k], NULL);
  free(tids);
  free(jobs);
}

float oracle_uniform_at(uint64_t seed, uint64_t idx) {
  return uniform_pm1(seed, idx);
}

/* fp64-accumulated reference rows R[r][j] = sum_k (double)A[r,k]*(double)B[k,j]
 * for r in rows[0..nrows); out is nrows x N. Row-major with leading dims. */
void oracle_sgemm_ref_rows(const float* A, const float* B, uint32_t N,
                           uint32_t K, uint32_t lda, uint32_t ldb,
                           const uint32_t* rows, uint32_t nrows, double* out) {
  for (uint32_t t = 0; t < nrows; ++t) {
    const float* a = A + (size_t)rows[t] * lda;
    double* o = out + (size_t)t * N;
    memset(o, 0, sizeof(double) * N);
    for (uint32_t k = 0; k < K; ++k) {
      double av = (double)a[k];
      const float* b = B + (size_t)k * ldb;
      for (uint32_t j = 0; j < N; ++j)
        o[j] += av * (double)b[j];
    }
  }
}

/* Normwise error of computed rows C (nrows x N, pitch ldc, rows taken from
 * C + rows[t]*ldc) against R: max over rows of max_j|C-R| / max_j|R|. */
double oracle_sgemm_rel_err(const float* C, uint32_t ldc, const double* R,
                            uint32_t N, const uint32_t* rows,
                            uint32_t nrows) {
  double worst = 0.0;
  for (uint32_t t = 0; t < nrows; ++t) {
    const float* c = C + (size_t)rows[t] * ldc;
    const double* r = R + (size_t)t * N;
    double num = 0.0, den = 0.0;
    for (uint32_t j = 0; j < N; ++j) {
      double d = (double)c[j] - r[j];
      if (d < 0) d = -d;
      double m = r[j] < 0 ? -r[j] : r[j];
      if (d > num) num = d;
      if (m > den) den = m;
    }
    double e = den > 0 ? num / den : num;
    if (e > worst) worst = e;
  }
  return worst;
}

/* ---- builder-authored CPU baseline: threaded, blocked fp32 ---------------
 * One worker per row block (the CPU analogue of one actor per row block);
 * the inner loop streams B rows so gcc vectorises it. */

typedef struct {
  const float* A;
  const float* B;
  float* C;
  uint32_t N, K, lda, ldb, ldc;
  uint32_t row_begin, row_end, row_step, block;
} gemm_job;

static void* gemm_worker(void* arg) {
  gemm_job* j = (gemm_job*)arg;
  const uint32_t KB = 256, NB = 1024;
  for (uint32_t r0 = j->row_begin; r0 < j->row_end; r0 += j->row_step) {
    uint32_t r1 = r0 + j->block;
    if (r1 > j->row_end) r1 = j->row_end;
    for (uint32_t r = r0; r < r1; ++r)
      memset(j->C + (size_t)r * j->ldc, 0, sizeof(float) * j->N);
    for (uint32_t n0 = 0; n0 < j->N; n0 += NB) {
      uint32_t n1 = n0 + NB < j->N ? n0 + NB : j->N;
      for (uint32_t k0 = 0; k0 < j->K; k0 += KB) {
        uint32_t k1 = k0 + KB < j->K ? k0 + KB : j->K;
        for (uint32_t r = r0; r < r1; ++r) {
          float* c = j->C + (size_t)r * j->ldc;
          const float* a = j->A + (size_t)r * j->lda;
          for (uint32_t k = k0; k < k1; ++k) {
            float av = a[k];
            const float* b = j->B + (size_t)k * j->ldb;
            for (uint32_t n = n0; n < n1; ++n)
              c[n] += av * b[n];
          }
        }
      }
    }
  }
  return NULL;
}

/* Computes rows [row_begin,row_end) of C = A*B (every `stride`-th row block
 * of `block` rows when sampling). */
void oracle_sgemm_f32_mt(const float* A, const float* B, float* C, uint32_t N,
                         uint32_t K, uint32_t lda, uint32_t ldb, uint32_t ldc,
                         uint32_t row_begin, uint32_t row_end, uint32_t block,
                         uint32_t threads) {
  if (threads == 0)
    threads = 1;
  if (block == 0)
    block = 16;
  pthread_t* tids = (pthread_t*)calloc(threads, sizeof(pthread_t));
  gemm_job* jobs = (gemm_job*)calloc(threads, sizeof(gemm_job));
  for (uint32_t t = 0; t < threads; ++t) {
    jobs[t] = (gemm_job){A, B, C, N, K, lda, ldb, ldc,
                         row_begin + t * block, row_end, threads * block,
                         block};
    pthread_create(&tids[t], NULL, gemm_worker, &jobs[t]);
  }
  for (uint32_t t = 0; t < threads; ++t)
    pthread_join(tids[t], NULL);
  free(tids);
  free(jobs);
}
