// Micro-benchmark (dev tool): instruction-mix variants of the keep-bit hash (bit-exactness is
// checked against the scalar reference form on every element).
#include <cstdio>
#include <cuda_runtime.h>
#include "rng_fast.cuh"
using namespace spl::rngk;

// x ^= x >> k with the high word's shift as IMAD.HI (FMA pipe) and the low word's as a funnel
// shift (ALU pipe): 3 ALU + 1 FMA instead of 4 ALU (xs_alu) or 2 ALU + 3 FMA (xs_fma)
__device__ __forceinline__ void xs_mix(uint32_t& lo, uint32_t& hi, int k, uint32_t m) {
  const uint32_t f = __funnelshift_r(lo, hi, k), g = __umulhi(hi, m);
  lo ^= f;
  hi ^= g;
}

template <int VAR>
__device__ __forceinline__ bool keep_var(uint32_t lo, uint32_t hi0, uint32_t hc, uint32_t mixed_lo,
                                         uint32_t mixed_hi, uint32_t t_lo, uint32_t t_hi,
                                         const ShiftMuls& sm, uint32_t c30 = 0) {
  if (VAR & 64) lo ^= c30; else lo ^= __funnelshift_r(lo, hi0, 30);
  uint32_t hi;
  {
    const uint64_t w = (uint64_t)lo * 0x1ce4e5b9u + ((uint64_t)hc << 32);
    hi = (uint32_t)(w >> 32) + lo * 0xbf58476du;
    lo = (uint32_t)w;
  }
  if (VAR & 256) xs_mix(lo, hi, 27, sm.m27); else if (VAR & 1) xs_alu(lo, hi, 27); else xs_fma(lo, hi, sm.m27);
  mul_c<0x133111ebu, 0x94d049bbu>(lo, hi);
  if (VAR & 32) {  // xor-shift 31 fused with ^ mix64(key) into 3-input LOP3s
    const uint32_t f = __funnelshift_r(lo, hi, 31), g = hi >> 31;
    lo = lo ^ f ^ mixed_lo;
    hi = hi ^ g ^ mixed_hi;
  } else {
    if (VAR & 256) xs_mix(lo, hi, 31, sm.m31); else if (VAR & 2) xs_alu(lo, hi, 31); else xs_fma(lo, hi, sm.m31);
    lo ^= mixed_lo;
    hi ^= mixed_hi;
  }
  if (VAR & 128) {  // + G as IMAD.WIDE.U32 (lo * one + G, FMA pipe) + one IADD for the high half
    const uint64_t w = (uint64_t)lo * sm.one + 0x9e3779b97f4a7c15ULL;
    hi = hi + (uint32_t)(w >> 32);
    lo = (uint32_t)w;
  } else {
    const uint64_t w = ((uint64_t)hi << 32 | lo) + 0x9e3779b97f4a7c15ULL;
    hi = (uint32_t)(w >> 32);
    lo = (uint32_t)w;
  }
  if (VAR & 256) xs_mix(lo, hi, 30, sm.m30); else if (VAR & 4) xs_fma(lo, hi, sm.m30); else xs_alu(lo, hi, 30);
  mul_c<0x1ce4e5b9u, 0xbf58476du>(lo, hi);
  if (VAR & 256) xs_mix(lo, hi, 27, sm.m27); else if (VAR & 8) xs_alu(lo, hi, 27); else xs_fma(lo, hi, sm.m27);
  mul_c<0x133111ebu, 0x94d049bbu>(lo, hi);
  if (VAR & 16) {  // high word decides unless equal to the threshold's
    const uint32_t h2 = hi ^ ((VAR & 512) ? __umulhi(hi, sm.m31) : (hi >> 31));
    if (__builtin_expect(h2 != t_hi, 1)) return h2 > t_hi;
    const uint32_t l2 = lo ^ __funnelshift_r(lo, hi, 31);
    return l2 >= t_lo;
  }
  xs_alu(lo, hi, 31);
  return (((uint64_t)hi << 32) | lo) >= (((uint64_t)t_hi << 32) | t_lo);
}

__device__ __forceinline__ bool keep_ref(uint64_t mixed, uint64_t tsh, uint64_t idx_cg) {
  return mix_post((mix_post(idx_cg) ^ mixed) + kG) >= tsh;
}

template <int VAR, int NT = 256, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) kb(uint64_t mixed, uint64_t tsh, int nrows, int W, int s,
                                          uint32_t* bits, ShiftMuls sm, int check, int* bad) {
  const uint32_t mixed_lo = (uint32_t)mixed, mixed_hi = (uint32_t)(mixed >> 32);
  const uint32_t t_lo = (uint32_t)tsh, t_hi = (uint32_t)(tsh >> 32);
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < nrows; row += warps) {
    const uint64_t base = (uint64_t)row * s + kC + kG;
    for (int w = lane; w < W; w += 32) {
      const uint64_t bw = base + 32u * w;
      const uint32_t blo = (uint32_t)bw, bhi = (uint32_t)(bw >> 32);
      uint32_t word = 0;
      if (blo <= 0xffffffffu - 31u) {
        const uint32_t hx = bhi ^ (bhi >> 30);
        const uint32_t hc = hx * 0x1ce4e5b9u;
        if ((VAR & 64) && (blo >> 30) == ((blo + 31u) >> 30)) {  // lo >> 30 constant in the word
          const uint32_t c30 = __funnelshift_r(blo, bhi, 30);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (keep_var<VAR>(blo + j, bhi, hc, mixed_lo, mixed_hi, t_lo, t_hi, sm, c30)) word |= 1u << j;
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (keep_var<VAR & ~64>(blo + j, bhi, hc, mixed_lo, mixed_hi, t_lo, t_hi, sm)) word |= 1u << j;
        }
      }
      if (check) {
        uint32_t ref = 0;
        for (int j = 0; j < 32; ++j) ref |= (keep_ref(mixed, tsh, bw + j) ? 1u : 0u) << j;
        if (ref != word && blo <= 0xffffffffu - 31u) atomicAdd(bad, 1);
      }
      bits[(int64_t)row * W + w] = word;
    }
  }
}

template <int VAR, int NT = 256, int MINB = 1>
void run(uint32_t* bits, int* bad, int nrows, int W, int s, int ctas_per_sm = 8) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  ShiftMuls sm{4u, 32u, 2u, 1u};
  const uint64_t mixed = 0x1234567890abcdefULL, tsh = 0x1999999999999800ULL;
  cudaMemset(bad, 0, 4);
  kb<VAR, NT, MINB><<<148 * 4, NT>>>(mixed, tsh, nrows / 64, W, s, bits, sm, 1, bad);
  int nb = 0;
  cudaMemcpy(&nb, bad, 4, cudaMemcpyDeviceToHost);
  const int grid = 148 * ctas_per_sm;
  kb<VAR, NT, MINB><<<grid, NT>>>(mixed, tsh, nrows, W, s, bits, sm, 0, bad);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) kb<VAR, NT, MINB><<<grid, NT>>>(mixed, tsh, nrows, W, s, bits, sm, 0, bad);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, kb<VAR, NT, MINB>);
  printf("VAR %3d NT %3d MINB %d ctas/SM %2d regs=%3d  %.3f ms  mismatches=%d\n", VAR, NT, MINB,
         ctas_per_sm, at.numRegs, ms / 5, nb);
}

int main() {
  const int s = 2048, nrows = 64 * 4 * 2048, W = s / 32;
  uint32_t* bits;
  int* bad;
  cudaMalloc(&bits, (size_t)nrows * W * 4);
  cudaMalloc(&bad, 4);
  for (int rep = 0; rep < 2; ++rep) {
    run<75 | 128 | 16, 1024, 1>(bits, bad, nrows, W, s, 1);          // production form
    run<75 | 128 | 16 | 256, 1024, 1>(bits, bad, nrows, W, s, 1);    // hi shifts as IMAD.HI
    run<75 | 128 | 16 | 256 | 512, 1024, 1>(bits, bad, nrows, W, s, 1);
    run<75 | 128 | 16 | 32 | 256, 1024, 1>(bits, bad, nrows, W, s, 1);
    run<75 | 128 | 16 | 32 | 256 | 512, 1024, 1>(bits, bad, nrows, W, s, 1);
    run<75 | 128 | 16 | 32, 1024, 1>(bits, bad, nrows, W, s, 1);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
