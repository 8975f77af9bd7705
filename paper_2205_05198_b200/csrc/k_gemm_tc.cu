// tcgen05 / TMEM / TMA bf16 GEMM for sm_100a (placeholder until the kernel lands).
#include "kernels.hpp"

namespace spl::k {
bool gemm_tc_supported(const GemmArgs&) { return false; }
void gemm_tc(const GemmArgs&, cudaStream_t) { raise(3, "tcgen05 gemm not built"); }
}  // namespace spl::k
