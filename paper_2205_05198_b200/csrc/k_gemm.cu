// GEMM dispatch: bf16 shapes the tcgen05 kernel can tile go to the tensor cores
// (k_gemm_tc.cu); fp32 (the exact-fp32 execution dtype) and unaligned shapes use the SIMT
// kernel (k_gemm_simt.cu). Both are on-device; there is no host path.
#include <atomic>
#include <cstdio>

#include "kernels.hpp"

namespace spl::k {

template <typename T>
void gemm_simt(const GemmArgs& a, cudaStream_t st);
bool gemm_tc_supported(const GemmArgs& a);
void gemm_tc(const GemmArgs& a, cudaStream_t st);

template <>
void gemm<float>(const GemmArgs& a, cudaStream_t st) {
  require(a.a_shards <= 1 && a.b_shards <= 1, "sharded GEMM operands need the tcgen05 path");
  gemm_simt<float>(a, st);
}
template <>
void gemm<bf16>(const GemmArgs& a, cudaStream_t st) {
  if (gemm_tc_supported(a)) gemm_tc(a, st);
  else {
    require(a.a_shards <= 1 && a.b_shards <= 1, "sharded GEMM operands need the tcgen05 path");
    // bf16 shapes off the tensor-core path (dimensions or leading dimensions not multiples of
    // 8 / 16-byte alignment): said once per process, so a slow layer is never silent
    static std::atomic<bool> told{false};
    if (!told.exchange(true))
      fprintf(stderr, "libspl: bf16 GEMM M=%lld N=%lld K=%lld (lda %lld, ldb %lld, ldc %lld) is not "
                      "tcgen05-aligned; using the SIMT kernel\n", (long long)a.M, (long long)a.N,
              (long long)a.K, (long long)a.lda, (long long)a.ldb, (long long)a.ldc);
    gemm_simt<bf16>(a, st);
  }
}
template <>
int gemm_backend<float>(const GemmArgs&) {
  return 0;
}
template <>
int gemm_backend<bf16>(const GemmArgs& a) {
  return gemm_tc_supported(a) ? 1 : 0;
}

}  // namespace spl::k
