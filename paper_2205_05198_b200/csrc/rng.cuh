// Device counter RNG, bit-exact with the reference's splitmix64 scheme
// (/root/reference/proj/core/src/seqpar/rng.cpp:22-45).
//
// keep(i) of the reference is `uniform01(folded, i) >= p`, i.e.
//   (double)(hash_counter(folded, i) >> 11) * 2^-53 >= p.
// Both sides are exact in double, so it equals the integer test
//   (hash >> 11) >= ceil(p * 2^53)
// which the kernels evaluate without any floating point. mix64(folded) is hoisted out of
// every loop (hash_counter = mix64(mix64(key) ^ mix64(i + C))).
#pragma once
#include <cmath>
#include <cstdint>

namespace spl {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t hash_counter(uint64_t key, uint64_t index) {
  return mix64(mix64(key) ^ mix64(index + 0x632be59bd9b4e019ULL));
}

inline uint64_t fold_mask_key(uint64_t seed, uint32_t layer, uint32_t op, uint32_t microbatch) {
  uint64_t k = mix64(seed);
  k = mix64(k ^ (uint64_t)layer);
  k = mix64(k ^ ((uint64_t)op << 20));
  k = mix64(k ^ ((uint64_t)microbatch << 40));
  return k;
}

// Dropout site ids of block.cpp:34.
enum MaskOp : uint32_t { kSoftmaxDrop = 0, kAttnOutDrop = 1, kMlpDrop = 2 };

struct DropKey {
  uint64_t mixed;   // mix64(folded key)
  uint64_t thresh;  // ceil(p * 2^53): keep iff (hash >> 11) >= thresh
  float inv_keep;   // 1 / (1 - p), rounded from the double of the reference
};

inline DropKey make_drop_key(uint64_t seed, uint32_t layer, uint32_t op, uint32_t microbatch,
                             double p) {
  DropKey k;
  k.mixed = mix64(fold_mask_key(seed, layer, op, microbatch));
  k.thresh = (uint64_t)std::ceil(p * 9007199254740992.0);  // exact: p*2^53 < 2^53
  k.inv_keep = (float)(1.0 / (1.0 - p));
  return k;
}

__device__ __forceinline__ bool drop_keep(const DropKey& k, uint64_t index) {
  return (mix64(k.mixed ^ mix64(index + 0x632be59bd9b4e019ULL)) >> 11) >= k.thresh;
}

}  // namespace spl
