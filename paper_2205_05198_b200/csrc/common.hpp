// Shared host/device definitions of libspl (B200 sequence-parallel layer).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace spl {

// Status-carrying exception; the C ABI maps it to the int codes of spl.h.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const std::string& msg) {
  if (!ok) raise(1, msg);
}

#define SPL_CUDA(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      ::spl::raise(3, std::string(#expr " failed: ") + cudaGetErrorString(e_) + " at " +  \
                          __FILE__ + ":" + std::to_string(__LINE__));                      \
  } while (0)

#define SPL_CHECK_LAUNCH() SPL_CUDA(cudaGetLastError())

enum class DType : int { F32 = 0, BF16 = 1 };
inline size_t dsize(DType t) { return t == DType::F32 ? 4 : 2; }

using bf16 = __nv_bfloat16;

__host__ __device__ inline float to_f(float v) { return v; }
__device__ inline float to_f(bf16 v) { return __bfloat162float(v); }
template <typename T> __device__ inline T from_f(float v);
template <> __device__ inline float from_f<float>(float v) { return v; }
template <> __device__ inline bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// Kernel classes for the per-class profiler (spl_profile_read).
enum KClass : int { K_GEMM = 0, K_ATTN = 1, K_ELEM = 2, K_COMM = 3, K_OTHER = 4, K_NCLASS = 5 };

constexpr int kNumSMs = 148;

// Message of the last failing C-ABI call on this thread (spl_last_error); defined in api.cu.
extern thread_local std::string g_last_error;

// Runs an extern "C" entry point body, mapping exceptions to the status codes of spl.h:
// spl::Error -> its code, std::invalid_argument -> SPL_EINVAL (1), std::domain_error ->
// SPL_EDOMAIN (2), anything else -> SPL_ECUDA (3).
template <typename F>
int c_guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return 0;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_last_error = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 3;
  }
}

}  // namespace spl
