// Exact-fp32 SIMT GEMM with the fused epilogues. This is the fp32 execution dtype's GEMM
// (the reference "tiny" config runs in fp32 for tight parity) and the
// kernel used for shapes the tcgen05 GEMM cannot tile (tiny/unaligned widths). bf16 GEMMs
// of aligned shapes go to the tcgen05/TMEM kernel in k_gemm_tc.cu.
#include "gemm_epilogue.cuh"

namespace spl::k {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_k(GemmArgs g) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const T* A = static_cast<const T*>(g.A);
  const T* B = static_cast<const T*>(g.B);
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int tid = threadIdx.x;
  const int tr = tid / 16, tc = tid % 16;
  const int64_t a_sm = g.amaj == Major::K ? g.lda : 1, a_sk = g.amaj == Major::K ? 1 : g.lda;
  const int64_t b_sk = g.bmaj == Major::K ? 1 : g.ldb, b_sn = g.bmaj == Major::K ? g.ldb : 1;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  for (int64_t k0 = 0; k0 < g.K; k0 += BK) {
    // 64x16 A tile and 16x64 B tile, 4 elements per thread each; the index order follows
    // the contiguous dimension of each operand so the loads coalesce.
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      int mm, kk;
      if (g.amaj == Major::K) { mm = idx / BK; kk = idx % BK; }
      else { kk = idx / BM; mm = idx % BM; }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < g.M && gk < g.K) ? to_f(A[gm * a_sm + gk * a_sk]) : 0.f;
      int nn, kb;
      if (g.bmaj == Major::K) { nn = idx / BK; kb = idx % BK; }
      else { kb = idx / BN; nn = idx % BN; }
      const int64_t gn = n0 + nn, gkb = k0 + kb;
      Bs[kb][nn] = (gn < g.N && gkb < g.K) ? to_f(B[gkb * b_sk + gn * b_sn]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][tr * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tc * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t m = m0 + tr * TM + i, n = n0 + tc * TN + j;
      if (m < g.M && n < g.N) epi_store<T>(g, m, n, acc[i][j]);
    }
}

}  // namespace

template <typename T>
void gemm_simt(const GemmArgs& a, cudaStream_t st) {
  if (a.M == 0 || a.N == 0) return;
  dim3 grid((unsigned)((a.N + BN - 1) / BN), (unsigned)((a.M + BM - 1) / BM));
  gemm_simt_k<T><<<grid, 256, 0, st>>>(a);
  SPL_CHECK_LAUNCH();
}

template void gemm_simt<float>(const GemmArgs&, cudaStream_t);
template void gemm_simt<bf16>(const GemmArgs&, cudaStream_t);

}  // namespace spl::k
