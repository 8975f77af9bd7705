// Fused GEMM epilogues shared by the SIMT and the tcgen05 GEMMs.
#pragma once
#include "kernels.hpp"

namespace spl::k {

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float gelu_erf_grad(float x) {
  const float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752f));
  const float pdf = 0.3989422804014327f * __expf(-0.5f * x * x);
  return cdf + x * pdf;
}

// Applies the epilogue to one accumulator value at (m, n).
template <typename T>
__device__ __forceinline__ void epi_store(const GemmArgs& g, int64_t m, int64_t n, float acc) {
  switch (g.epi) {
    case Epi::Store:
      gemm_row<T>(g, m)[n] = from_f<T>(acc);
      break;
    case Epi::Bias:
      gemm_row<T>(g, m)[n] = from_f<T>(acc + g.bias[n]);
      break;
    case Epi::BiasGelu: {
      const T pre = from_f<T>(acc + g.bias[n]);
      gemm_row<T>(g, m)[n] = pre;
      static_cast<T*>(g.C2)[m * g.ldc + n] = from_f<T>(gelu_erf(to_f(pre)));
      break;
    }
    case Epi::GeluBwd: {
      const float x = to_f(static_cast<const T*>(g.aux)[m * g.ldaux + n]);
      gemm_row<T>(g, m)[n] = from_f<T>(acc * gelu_erf_grad(x));
      break;
    }
    case Epi::F32:
      gemm_row<float>(g, m)[n] = g.accumulate ? gemm_row<float>(g, m)[n] + acc : acc;
      break;
  }
}

}  // namespace spl::k
