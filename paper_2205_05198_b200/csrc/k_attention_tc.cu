// Tensor-core attention for bf16 (placeholder until the kernel lands).
#include "kernels.hpp"

namespace spl::k {
template <typename T>
bool attn_tc_supported(const AttnArgs& a);
template <typename T>
void attn_fwd_tc(const AttnArgs& a, cudaStream_t st);
template <typename T>
void attn_bwd_tc(const AttnArgs& a, const void* dout, void* dqkv, float* delta, cudaStream_t st);
template <>
bool attn_tc_supported<bf16>(const AttnArgs&) { return false; }
template <>
void attn_fwd_tc<bf16>(const AttnArgs&, cudaStream_t) {}
template <>
void attn_bwd_tc<bf16>(const AttnArgs&, const void*, void*, float*, cudaStream_t) {}
}  // namespace spl::k
