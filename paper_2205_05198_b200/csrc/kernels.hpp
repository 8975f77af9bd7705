// Launchers of the sm_100a kernels of libspl. Every launcher is asynchronous on `st`.
#pragma once
#include <cstdint>

#include "common.hpp"
#include "rng.cuh"

namespace spl::k {

// tensor-parallel ranks a fused reduce-scatter addresses (the local-rank limit of LocalComm)
constexpr int kMaxScatterRanks = 16;


// ---------------------------------------------------------------- parameters
// LayerParams::random on the device (block.cpp:234-265): out[i, j] (ld_out) =
//   lo + (hi - lo) * uniform01(key, (row0 + i) * ld_full + col0 + j) + add
// evaluated in fp64 without contraction, then rounded once to T.
template <typename T>
void init_uniform(T* out, int64_t rows, int64_t cols, int64_t ld_out, int64_t row0,
                  int64_t col0, int64_t ld_full, uint64_t key, double lo, double hi, double add,
                  cudaStream_t st);

// ---------------------------------------------------------------- elementwise / row ops
// y = LayerNorm(x) with fp32 two-pass statistics (block.cpp:300-328); saves mean, rstd.
template <typename T>
void layernorm_fwd(const T* x, const float* gain, const float* bias, T* y, float* mean,
                   float* rstd, int64_t rows, int64_t h, float eps, cudaStream_t st);

// Bias-dropout-residual (block.cpp:568-578 / 589-600):
//   r = resid + keep(base + i) * (a + bias) / (1 - p), mask[i] = keep
// and, when ln_out != nullptr, ln_out = LayerNorm(r) with saved stats (the LN2 fusion).
// nonfinite (optional) is OR-ed with 1 when any r is not finite.
template <typename T>
void bias_dropout_residual(const T* a, const float* bias, const T* resid, T* r_out,
                           uint8_t* mask_out, T* ln_out, const float* gain, const float* lnb,
                           float* mean, float* rstd, int64_t rows, int64_t h, DropKey key,
                           uint64_t base_index, float eps, int* nonfinite, cudaStream_t st);

// ---- consumer side of the reduce-scatter fused into a row-parallel GEMM (GemmArgs::scatter):
// the t landing slots of this rank, summed in rank order 0..t-1 in fp32 and rounded to T
// (collectives.cpp:40-46), after waiting until all t sources signalled past the generation.
struct SlotSrc {
  const void* p[kMaxScatterRanks] = {};
  int n = 0;
  const uint32_t* flags = nullptr;  // t arrival counters (this rank)
  const uint32_t* gen = nullptr;    // this rank's generation counter
};
struct FlagPtrs {
  uint32_t* p[kMaxScatterRanks] = {};
  int n = 0;
};
// source side, after its GEMM: system-scope release increment of every destination's counter
void p2p_signal(const FlagPtrs& f, cudaStream_t st);
// destination side, after its consumer: generation += 1
void p2p_advance(uint32_t* gen, cudaStream_t st);
// BDR(+LN) whose input partial is the sum of the slots (the forward's ḡ + 568-578 / 588-600)
template <typename T>
void bias_dropout_residual_slots(const SlotSrc& a, const float* bias, const T* resid, T* r_out,
                                 uint8_t* mask_out, T* ln_out, const float* gain, const float* lnb,
                                 float* mean, float* rstd, int64_t rows, int64_t h, DropKey key,
                                 uint64_t base_index, float eps, int* nonfinite, cudaStream_t st);
// out[n] = rank-ordered sum of the slots (the backward's g-dual reduce-scatters)
template <typename T>
void reduce_slots(const SlotSrc& a, T* out, int64_t n, cudaStream_t st);

// out = dy * mask / (1 - p) (block.cpp:77-79) and per-chunk column sums of out (the bias
// gradient, tensor.cpp:109-114) into partials[chunk][h].
template <typename T>
void dropout_bwd_colsum(const T* dy, const uint8_t* mask, float inv_keep, T* out,
                        float* partials, int64_t rows, int64_t h, int chunk_rows,
                        cudaStream_t st);

// dx = resid_grad + LayerNormBackward(dy) (block.cpp:330-360 + the residual add at 678/723),
// with per-chunk partial column sums of dy*xhat (gain grad) and dy (bias grad).
template <typename T>
void layernorm_bwd(const T* dy, const T* x, const float* mean, const float* rstd,
                   const float* gain, const T* resid_grad, T* dx, float* pgain, float* pbias,
                   int64_t rows, int64_t h, int chunk_rows, cudaStream_t st);

// partials[chunk][j] = sum_{rows of chunk} x[r * ld + j], j < n.
template <typename T>
void colsum_partial(const T* x, int64_t rows, int64_t n, int64_t ld, float* partials,
                    int chunk_rows, cudaStream_t st);
// out[j] (+)= sum_c partials[c][j], chunks summed in order (deterministic).
void reduce_partials(const float* partials, int nchunks, int64_t n, float* out, bool accumulate,
                     cudaStream_t st);
inline int num_chunks(int64_t rows, int chunk_rows) {
  return (int)((rows + chunk_rows - 1) / chunk_rows);
}

// ---------------------------------------------------------------- collectives (local ranks)
// out[i] = sum_{r=0..nparts-1} parts[r][offset + i] in rank order, fp32 accumulation
// (the ordered_sum of collectives.cpp:40-46); parts is a DEVICE array of pointers.
template <typename T>
void ordered_sum(const T* const* parts_dev, int nparts, int64_t offset, int64_t n, T* out,
                 cudaStream_t st);
void ordered_sum_f32(const float* const* parts_dev, int nparts, int64_t n, float* out,
                     cudaStream_t st);

// ---------------------------------------------------------------- casts
template <typename T>
void cast_to_f64(const T* in, double* out, int64_t n, cudaStream_t st);
void u8_to_f64(const uint8_t* in, double* out, int64_t n, cudaStream_t st);
void f32_to_f64(const float* in, double* out, int64_t n, cudaStream_t st);

// ---------------------------------------------------------------- GEMM
// C[M,N] = A[M,K] · B[K,N] with fp32 accumulation and a fused epilogue.
// A(m,k) = A[m*lda + k] (Major::K) or A[k*lda + m] (Major::MN);
// B(k,n) = B[n*ldb + k] (Major::K) or B[k*ldb + n] (Major::MN).
enum class Major : int { K = 0, MN = 1 };
enum class Epi : int {
  Store = 0,     // C = acc                                (T)
  Bias = 1,      // C = acc + bias[n]                      (T)
  BiasGelu = 2,  // C = acc + bias[n]; C2 = gelu_erf(C)    (T, T) — FC1 (block.cpp:584-585)
  GeluBwd = 3,   // C = acc * gelu'(aux[m,n])              (T)    — FC2 dgrad (block.cpp:660-662)
  F32 = 4,       // Cf = acc                               (fp32) — weight gradients
};
struct GemmArgs {
  int64_t M = 0, N = 0, K = 0;
  const void* A = nullptr;
  int64_t lda = 0;
  Major amaj = Major::K;
  const void* B = nullptr;
  int64_t ldb = 0;
  Major bmaj = Major::K;
  void* C = nullptr;
  int64_t ldc = 0;
  Epi epi = Epi::Store;
  const float* bias = nullptr;
  void* C2 = nullptr;       // BiasGelu second output (ldc)
  const void* aux = nullptr;  // GeluBwd pre-activation (ld = ldaux)
  int64_t ldaux = 0;
  // Row scatter (the reduce-scatter fused into a row-parallel GEMM): when scatter_n > 0, row m
  // of C is written to scatter[m / scatter_rows] + (m % scatter_rows) * ldc instead of
  // C + m * ldc — i.e. into the landing slot this rank owns in the buffer of the rank that
  // holds that sequence shard (peer memory over NVLink, or a local buffer for simulated ranks).
  static constexpr int kMaxScatter = kMaxScatterRanks;
  void* scatter[kMaxScatter] = {};
  int scatter_n = 0;
  int64_t scatter_rows = 0;
  int accumulate = 0;  // Epi::F32 only: C += A·B (gradient accumulation across microbatches)
  // Sharded operand (the all-gather fused into the GEMM): when a_shards > 1, A's token
  // dimension (M for Major::K, K for Major::MN) is split into a_shards row blocks of shard_rows
  // rows, block q at a_shard[q] (leading dimension lda); likewise B (Major::MN: along K). The
  // TMA producer of the CTA-pair kernel picks the block of each tile, so no gathered copy exists.
  static constexpr int kMaxShards = 8;
  const void* a_shard[kMaxShards] = {};
  const void* b_shard[kMaxShards] = {};
  int a_shards = 0, b_shards = 0;
  int64_t shard_rows = 0;
};
// Base of output row m of a GEMM (honours the row scatter).
template <typename U>
__host__ __device__ inline U* gemm_row(const GemmArgs& g, int64_t m) {
  if (g.scatter_n > 0) {
    const int64_t q = m / g.scatter_rows;
    return static_cast<U*>(g.scatter[q]) + (m - q * g.scatter_rows) * g.ldc;
  }
  return static_cast<U*>(g.C) + m * g.ldc;
}
template <typename T>
void gemm(const GemmArgs& a, cudaStream_t st);
// Which implementation gemm<T> used for these args (for the profiler): 1 = tcgen05.
template <typename T>
int gemm_backend(const GemmArgs& a);
// True when a bf16 GEMM of these arguments runs on the CTA-pair tcgen05 kernel (the only one
// that takes sharded operands).
bool gemm_tc_pair_path(const GemmArgs& a);

// ---------------------------------------------------------------- attention
// Q/K/V packed in one [s*b, ld] buffer: row = s_i*b + b_j; Q cols [qoff + hl*hd, +hd),
// K at koff, V at voff. O: [s*b, ldo], head hl at column hl*hd.
struct AttnArgs {
  int64_t s = 0, b = 0, lh = 0, hd = 0;
  int64_t head_offset = 0, heads_total = 0;  // global head index = head_offset + hl
  const void* qkv = nullptr;
  int64_t ld = 0, qoff = 0, koff = 0, voff = 0;
  void* o = nullptr;
  int64_t ldo = 0;
  float scale = 1.f;
  int causal = 0;
  DropKey drop{};
  float* lse = nullptr;  // [lh, b, s] natural-log sum-exp of the scaled scores
  // stored interior (no-recompute regime): {lh, b, s, s}
  void* sm = nullptr;
  uint8_t* mask = nullptr;
  void* sd = nullptr;
  // softmax-dropout keep bits [lh*b*s][ceil(s/32)] from attn_keep_bits (bf16 tensor-core path);
  // a transient buffer refilled before each attention forward and backward.
  uint32_t* keepbits = nullptr;
  int masked_only = 0;  // backward: 1 = every tile through the per-element validity path (A/B)
  int stats_shfl = 0;   // dK/dV: 1 = per-element shuffles for row stats / keep bits (A/B)
  // fused backward (attn_bwd_fused): fp32 dQ accumulator [lh*b][s][hd] and the per-row
  // statistics [2][lh*b*s] (-lse·log2 e, -rowdot); transient workspaces
  float* dq_acc = nullptr;
  float* bstat = nullptr;
  // keep bits in the transposed layout [lh*b][s/32][s] (word = one key x 32 queries), filled by
  // attn_keep_bits for and read by the fused backward; else [lh*b*s][ceil(s/32)]
  int keep_t = 0;
};
inline int64_t keepbits_words(int64_t lh, int64_t b, int64_t s) { return lh * b * s * ((s + 31) / 32); }
// Forward. If a.sm != nullptr the interior is materialised (softmax_out, mask, dropout_out).
template <typename T>
void attn_fwd(const AttnArgs& a, cudaStream_t st);
// Backward: dO [s*b, ldo] (same layout as O) -> dQ/dK/dV into dqkv (same layout as qkv).
// Recomputes P and the dropout mask from Q, K, lse and the counter RNG (selective), or reads
// the stored interior when a.sm != nullptr (no-recompute). delta: [lh*b*s] fp32 scratch.
template <typename T>
void attn_bwd(const AttnArgs& a, const void* dout, void* dqkv, float* delta, cudaStream_t st);
// The counter-RNG pass alone: fills a.keepbits (data-independent; may run on a side stream).
void attn_keep_bits(const AttnArgs& a, cudaStream_t st);
// tcgen05/TMEM forward (bf16, head_dim 64/96/128/160; recompute regimes single-pass, the
// no-recompute regime writes the stored interior); used by attn_fwd<bf16>.
bool attn_fwd_umma_supported(const AttnArgs& a);
void attn_fwd_umma(const AttnArgs& a, cudaStream_t st);
// Recompute-regime forward with two query tiles per CTA in ping-pong (k_attention_fwd_pp.cu);
// attn_fwd_umma dispatches to it when supported (SPL_ATTN_FWD_PP=0: off).
bool attn_fwd_pp_supported(const AttnArgs& a);
void attn_fwd_pp(const AttnArgs& a, cudaStream_t st);
// tcgen05/TMEM backward (recompute regimes: keep bits from attn_keep_bits; no-recompute: the
// stored interior). delta = rowdot(dO, O) must be computed first.
bool attn_bwd_umma_supported(const AttnArgs& a);
void attn_bwd_umma(const AttnArgs& a, const void* dout, void* dqkv, const float* delta,
                   cudaStream_t st);
// One-kernel backward (dK, dV and dQ from one recomputation; dQ summed over key blocks in an
// fp32 L2 accumulator): recompute regimes, bf16, head_dim 64/96, s % 128 == 0, workspaces set.
// SPL_ATTN_DETERMINISTIC=1 turns it off (split kernels, bit-reproducible dQ).
bool attn_bwd_fused_supported(const AttnArgs& a);
// Whether attn_bwd<bf16> takes the fused path for these arguments (the layer fills the
// backward's keep bits in the transposed layout exactly when it does).
bool attn_bwd_uses_fused(const AttnArgs& a);
void attn_bwd_fused(const AttnArgs& a, const void* dout, void* dqkv, cudaStream_t st);

}  // namespace spl::k
