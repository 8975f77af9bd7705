/* fp64 GEMM for the oracle (TEST INFRASTRUCTURE — see oracle.h).
 * Stands in for the reference's Eigen3 products (tensor.cpp:57-107, block.cpp:148-149,
 * 179-189, 400-401). Generic strides cover matmul, matmul_transposed_rhs/lhs and the strided
 * per-head views. Each C element is accumulated sequentially over k (k = 0..K-1) whatever
 * the blocking or thread count, so results are deterministic and independent of the M/N
 * partitioning — the property the reference's t=1 bit-identity check relies on.
 * Blocked + packed with an AVX2/FMA 4x8 micro-kernel and OpenMP over output tiles. */
#include <immintrin.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "orc_internal.h"

#define MR 4
#define NR 8
#define MC 128
#define NC 256
#define KC 256

static int g_threads = 0;

int orc_set_threads(int n) {
#ifdef _OPENMP
  g_threads = n > 0 ? n : omp_get_max_threads();
  return g_threads;
#else
  (void)n;
  g_threads = 1;
  return 1;
#endif
}

int orc_threads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}

__attribute__((target("avx2,fma"))) static void micro_4x8(int64_t kc, const double* ap,
                                                          const double* bp, double* acc) {
  __m256d c00 = _mm256_loadu_pd(acc + 0), c01 = _mm256_loadu_pd(acc + 4);
  __m256d c10 = _mm256_loadu_pd(acc + 8), c11 = _mm256_loadu_pd(acc + 12);
  __m256d c20 = _mm256_loadu_pd(acc + 16), c21 = _mm256_loadu_pd(acc + 20);
  __m256d c30 = _mm256_loadu_pd(acc + 24), c31 = _mm256_loadu_pd(acc + 28);
  for (int64_t k = 0; k < kc; ++k) {
    const __m256d b0 = _mm256_loadu_pd(bp + k * NR);
    const __m256d b1 = _mm256_loadu_pd(bp + k * NR + 4);
    __m256d a = _mm256_broadcast_sd(ap + k * MR + 0);
    c00 = _mm256_fmadd_pd(a, b0, c00);
    c01 = _mm256_fmadd_pd(a, b1, c01);
    a = _mm256_broadcast_sd(ap + k * MR + 1);
    c10 = _mm256_fmadd_pd(a, b0, c10);
    c11 = _mm256_fmadd_pd(a, b1, c11);
    a = _mm256_broadcast_sd(ap + k * MR + 2);
    c20 = _mm256_fmadd_pd(a, b0, c20);
    c21 = _mm256_fmadd_pd(a, b1, c21);
    a = _mm256_broadcast_sd(ap + k * MR + 3);
    c30 = _mm256_fmadd_pd(a, b0, c30);
    c31 = _mm256_fmadd_pd(a, b1, c31);
  }
  _mm256_storeu_pd(acc + 0, c00);
  _mm256_storeu_pd(acc + 4, c01);
  _mm256_storeu_pd(acc + 8, c10);
  _mm256_storeu_pd(acc + 12, c11);
  _mm256_storeu_pd(acc + 16, c20);
  _mm256_storeu_pd(acc + 20, c21);
  _mm256_storeu_pd(acc + 24, c30);
  _mm256_storeu_pd(acc + 28, c31);
}

/* One MC x NC output tile, full K. */
static void gemm_tile(int64_t i0, int64_t mc, int64_t j0, int64_t nc, int64_t K, const double* a,
                      int64_t ars, int64_t acs, const double* b, int64_t brs, int64_t bcs,
                      double* c, int64_t ldc, int accumulate, double* apack, double* bpack) {
  const int64_t mp = (mc + MR - 1) / MR, np = (nc + NR - 1) / NR;
  for (int64_t k0 = 0; k0 < K; k0 += KC) {
    const int64_t kc = K - k0 < KC ? K - k0 : KC;
    for (int64_t p = 0; p < mp; ++p)
      for (int64_t k = 0; k < kc; ++k)
        for (int r = 0; r < MR; ++r) {
          const int64_t i = p * MR + r;
          apack[(p * kc + k) * MR + r] = i < mc ? a[(i0 + i) * ars + (k0 + k) * acs] : 0.0;
        }
    for (int64_t q = 0; q < np; ++q)
      for (int64_t k = 0; k < kc; ++k)
        for (int cc = 0; cc < NR; ++cc) {
          const int64_t j = q * NR + cc;
          bpack[(q * kc + k) * NR + cc] = j < nc ? b[(k0 + k) * brs + (j0 + j) * bcs] : 0.0;
        }
    for (int64_t p = 0; p < mp; ++p)
      for (int64_t q = 0; q < np; ++q) {
        double acc[MR * NR];
        const int64_t ib = p * MR, jb = q * NR;
        const int load = k0 > 0 || accumulate;
        for (int r = 0; r < MR; ++r)
          for (int cc = 0; cc < NR; ++cc) {
            const int64_t i = ib + r, j = jb + cc;
            acc[r * NR + cc] = (load && i < mc && j < nc) ? c[(i0 + i) * ldc + j0 + j] : 0.0;
          }
        micro_4x8(kc, apack + p * kc * MR, bpack + q * kc * NR, acc);
        for (int r = 0; r < MR; ++r)
          for (int cc = 0; cc < NR; ++cc) {
            const int64_t i = ib + r, j = jb + cc;
            if (i < mc && j < nc) c[(i0 + i) * ldc + j0 + j] = acc[r * NR + cc];
          }
      }
  }
}

void orc_gemm(int64_t M, int64_t N, int64_t K, const double* a, int64_t ars, int64_t acs,
              const double* b, int64_t brs, int64_t bcs, double* c, int64_t ldc, int accumulate) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    if (!accumulate)
      for (int64_t i = 0; i < M; ++i) memset(c + i * ldc, 0, sizeof(double) * (size_t)N);
    return;
  }
  const int64_t tm = (M + MC - 1) / MC, tn = (N + NC - 1) / NC, tiles = tm * tn;
  const int nthreads = orc_threads();
  const int64_t flops = M * N * K;
#pragma omp parallel num_threads(nthreads) if (tiles > 1 && flops > (1 << 20))
  {
    double* apack = (double*)aligned_alloc(64, sizeof(double) * MC * KC);
    double* bpack = (double*)aligned_alloc(64, sizeof(double) * NC * KC);
#pragma omp for schedule(dynamic, 1)
    for (int64_t tile = 0; tile < tiles; ++tile) {
      const int64_t ti = tile / tn, tj = tile % tn;
      const int64_t i0 = ti * MC, j0 = tj * NC;
      const int64_t mc = M - i0 < MC ? M - i0 : MC, nc = N - j0 < NC ? N - j0 : NC;
      gemm_tile(i0, mc, j0, nc, K, a, ars, acs, b, brs, bcs, c, ldc, accumulate, apack, bpack);
    }
    free(apack);
    free(bpack);
  }
}
