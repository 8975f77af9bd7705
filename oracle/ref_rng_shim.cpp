// Shim that lets the reference rng.cpp (compiled unmodified from /root/reference) link
// without tensor.cpp (which needs Eigen3, absent here), plus a C entry layer for ctypes.
// TEST INFRASTRUCTURE: used only to generate tests/golden/rng_kat.json and to cross-check
// the oracle's RNG restatement. The reference sources are compiled in place, never copied.
#include <cstdint>
#include <cstring>
#include <vector>

#include "actplan/seqpar/rng.hpp"
#include "actplan/seqpar/tensor.hpp"

namespace actplan::seqpar {
// Minimal definition of the one Tensor member rng.cpp needs (declared at tensor.hpp:29).
Tensor::Tensor(std::vector<std::int64_t> shape) : shape_(std::move(shape)) {
  std::int64_t n = 1;
  for (auto d : shape_) n *= d;
  data_.assign(static_cast<std::size_t>(n), 0.0);
}
}  // namespace actplan::seqpar

using namespace actplan::seqpar;

extern "C" {
std::uint64_t ref_hash_counter(std::uint64_t key, std::uint64_t index) {
  return hash_counter(key, index);
}
double ref_uniform01(std::uint64_t key, std::uint64_t index) { return uniform01(key, index); }
std::uint64_t ref_mask_key_fold(std::uint64_t seed, std::uint32_t layer, std::uint32_t op,
                                std::uint32_t microbatch) {
  MaskKey k{seed, layer, op, microbatch};
  return k.fold();
}
void ref_random_uniform(std::uint64_t key, std::int64_t n, double lo, double hi, double* out) {
  Tensor t = random_uniform(key, {n}, lo, hi);
  std::memcpy(out, t.data(), sizeof(double) * static_cast<std::size_t>(n));
}
int ref_dropout_mask(std::uint64_t seed, std::uint32_t layer, std::uint32_t op,
                     std::uint32_t microbatch, std::int64_t n, double p, double* out) {
  try {
    Tensor t = dropout_mask(MaskKey{seed, layer, op, microbatch}, {n}, p);
    std::memcpy(out, t.data(), sizeof(double) * static_cast<std::size_t>(n));
    return 0;
  } catch (...) {
    return 1;
  }
}
}
