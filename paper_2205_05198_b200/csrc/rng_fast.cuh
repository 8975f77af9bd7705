// Counter-RNG hot-loop forms shared by the kernels that generate dropout keep bits in bulk
// (the softmax-dropout keep-bit pass and the fused bias-dropout-residual kernels).
// Bit-exact with the reference's splitmix64 scheme (rng.cpp:22-45); see rng.cuh.
#pragma once
#include <cstdint>

#include "rng.cuh"

namespace spl::rngk {

// ---------------------------------------------------------------- counter RNG, hot-loop form
// keep(i) = (hash_counter(folded, i) >> 11) >= ceil(p*2^53)  (rng.cpp:31-37, block.cpp:63)
//   hash_counter(k, i) = mix64(mix64(k) ^ mix64(i + C)),  mix64(x) = post(x + G)
// With base = row_index*s + C + G precomputed per row, one element costs
//   post(base + key) ^ mixed, + G, post, 64-bit compare against thresh << 11.
constexpr uint64_t kG = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kC = 0x632be59bd9b4e019ULL;
// x * C mod 2^64 in three 32-bit multiplies (IMAD.WIDE + 2 IMAD)
template <uint64_t C>
__device__ __forceinline__ uint64_t mulc(uint64_t x) {
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
  const uint64_t w = (uint64_t)xl * (uint32_t)C;
  const uint32_t hi = (uint32_t)(w >> 32) + xl * (uint32_t)(C >> 32) + xh * (uint32_t)C;
  return ((uint64_t)hi << 32) | (uint32_t)w;
}
__device__ __forceinline__ uint64_t mix_post(uint64_t x) {
  x = mulc<0xbf58476d1ce4e5b9ULL>(x ^ (x >> 30));
  x = mulc<0x94d049bb133111ebULL>(x ^ (x >> 27));
  return x ^ (x >> 31);
}

struct ShiftMuls {
  uint32_t m30, m27, m31;  // 2^(32-k)
  uint32_t one;            // 1: the 64-bit "+ G" as IMAD.WIDE (FMA pipe) instead of IADD3 pairs
};
template <uint32_t CL, uint32_t CH>
__device__ __forceinline__ void mul_c(uint32_t& lo, uint32_t& hi) {  // (hi:lo) *= (CH:CL)
  const uint64_t w = (uint64_t)lo * CL;
  hi = (uint32_t)(w >> 32) + lo * CH + hi * CL;
  lo = (uint32_t)w;
}
__device__ __forceinline__ void xs_alu(uint32_t& lo, uint32_t& hi, int k) {  // x ^= x >> k
  lo ^= __funnelshift_r(lo, hi, k);
  hi ^= hi >> k;
}
__device__ __forceinline__ void xs_fma(uint32_t& lo, uint32_t& hi, uint32_t m) {  // m = 2^(32-k)
  const uint32_t a = __umulhi(lo, m), b = hi * m, c = __umulhi(hi, m);
  lo = lo ^ a ^ b;
  hi ^= c;
}
// C30: the caller guarantees lo >> 30 is the same for every key of the word, so the low half
// of the first xor-shift is a word constant: c30 = funnelshift_r(lo, hi0, 30) (one op per key
// saved, 2.3 % of the pass; tools/micro/bench_rng2.cu).
template <bool C30 = false>
__device__ __forceinline__ bool keep_fast(uint32_t lo, uint32_t hi0, uint32_t hc,
                                          uint32_t hi_xs, uint32_t mixed_lo, uint32_t mixed_hi,
                                          uint32_t t_lo, uint32_t t_hi, const ShiftMuls& sm,
                                          uint32_t c30 = 0) {
  // first mix_post; the high half (hi0) is loop-invariant: hi_xs = hi0 ^ (hi0 >> 30) and
  // hc = hi_xs * 0x1ce4e5b9 are precomputed per 32-key word.
  if constexpr (C30) lo ^= c30;
  else lo ^= __funnelshift_r(lo, hi0, 30);
  uint32_t hi;
  {
    const uint64_t w = (uint64_t)lo * 0x1ce4e5b9u + ((uint64_t)hc << 32);
    hi = (uint32_t)(w >> 32) + lo * 0xbf58476du;
    lo = (uint32_t)w;
  }
  (void)hi_xs;
  // Every xor-shift in funnel-shift (ALU) form: measured fastest on B200 (tools/micro/
  // bench_rng2.cu: 1.97 ms vs 2.12 ms for three in IMAD.HI form, 1.07e9 keys).
  xs_alu(lo, hi, 27);
  mul_c<0x133111ebu, 0x94d049bbu>(lo, hi);
  xs_alu(lo, hi, 31);
  // ^ mix64(key), + G (64-bit add as IMAD.WIDE with a 64-bit addend)
  lo ^= mixed_lo;
  hi ^= mixed_hi;
  {  // 64-bit + G as IMAD.WIDE.U32 (lo * sm.one + G: moves an ALU op to the FMA pipe)
    const uint64_t w = (uint64_t)lo * sm.one + 0x9e3779b97f4a7c15ULL;
    hi = hi + (uint32_t)(w >> 32);
    lo = (uint32_t)w;
  }
  xs_alu(lo, hi, 30);
  mul_c<0x1ce4e5b9u, 0xbf58476du>(lo, hi);
  xs_alu(lo, hi, 27);
  mul_c<0x133111ebu, 0x94d049bbu>(lo, hi);
  xs_alu(lo, hi, 31);
  return (((uint64_t)hi << 32) | lo) >= (((uint64_t)t_hi << 32) | t_lo);
}

// High word of the final hash only (keep_fast without its last low-word xor-shift and 64-bit
// compare): keep = hf > t_hi, or hf == t_hi and the low word >= t_lo. A tie has probability
// 2^-32 per key; the caller flags it (one predicate-OR compare) and redoes that word with
// keep_fast. Saves two of the ~44 integer instructions per key.
// RAW: the high word before the final xor-shift (hf = raw ^ (raw >> 31) differs from raw in
// bit 0 only), for callers that compare against the threshold on raw and fall back on the
// rare keys whose raw agrees with the threshold above bit 0.
template <bool C30 = false, bool RAW = false>
__device__ __forceinline__ uint32_t hash_hi(uint32_t lo, uint32_t hi0, uint32_t hc,
                                            uint32_t mixed_lo, uint32_t mixed_hi,
                                            const ShiftMuls& sm, uint32_t c30 = 0) {
  if constexpr (C30) lo ^= c30;
  else lo ^= __funnelshift_r(lo, hi0, 30);
  uint32_t hi;
  {
    const uint64_t w = (uint64_t)lo * 0x1ce4e5b9u + ((uint64_t)hc << 32);
    hi = (uint32_t)(w >> 32) + lo * 0xbf58476du;
    lo = (uint32_t)w;
  }
  xs_alu(lo, hi, 27);
  mul_c<0x133111ebu, 0x94d049bbu>(lo, hi);
  xs_alu(lo, hi, 31);
  lo ^= mixed_lo;
  hi ^= mixed_hi;
  {
    const uint64_t w = (uint64_t)lo * sm.one + 0x9e3779b97f4a7c15ULL;
    hi = hi + (uint32_t)(w >> 32);
    lo = (uint32_t)w;
  }
  xs_alu(lo, hi, 30);
  mul_c<0x1ce4e5b9u, 0xbf58476du>(lo, hi);
  xs_alu(lo, hi, 27);
  hi = __umulhi(lo, 0x133111ebu) + lo * 0x94d049bbu + hi * 0x133111ebu;
  return RAW ? hi : hi ^ (hi >> 31);
}

}  // namespace spl::rngk
