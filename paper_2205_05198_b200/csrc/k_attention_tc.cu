// bf16 attention core on tensor cores (mma.sync m16n8k16, fp32 accumulate), flash-style:
// the s×s interior never reaches HBM in the selective-recompute regime.
//
// Forward  fa_fwd:     per (64-query block, head, batch) CTA, 4 warps × 16 query rows; streams
//                      64-key K/V tiles (cp.async double buffer), online softmax in the log2
//                      domain, dropout keep bits from the counter RNG at the global {a,b,s,s}
//                      index (bit-exact with rng.cpp), O and the row LSE written at the end.
// Backward fa_bwd_dkdv: per 64-key CTA, loops over 32-query tiles recomputing Sᵀ = K Qᵀ,
//                      Pᵀ = exp(Sᵀ - LSE), keepᵀ, dPᵀ = V dOᵀ; accumulates dV += P̃ᵀ dO and
//                      dK += dSᵀ Q in registers (deterministic, no atomics).
//          fa_bwd_dq:  per 64-query CTA, loops over 32-key tiles: S, P, keep, dP = dO Vᵀ,
//                      dQ += dS K.
// rowdot_i = dO_i·O_i replaces Σ_j dSM_ij SM_ij of block.cpp:183 (algebraically equal).
#include <cstdlib>
#include <type_traits>

#include "kernels.hpp"
#include "rng_fast.cuh"

namespace spl::k {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// 16-byte async copy, zero-filled when !valid.
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Load `rows` rows (sequence positions r0..r0+rows-1 of head column col) into smem [rows][HD+8].
template <int HD, int ROWS, int NT>
__device__ __forceinline__ void load_tile(bf16* sm, const bf16* base, int64_t r0, int64_t s,
                                          int64_t rstride, int64_t col) {
  constexpr int CPR = HD / 8;  // 16B chunks per row
  for (int c = threadIdx.x; c < ROWS * CPR; c += NT) {
    const int r = c / CPR, k = c % CPR;
    const int64_t gr = r0 + r;
    const bool ok = gr < s;
    const bf16* src = base + (ok ? gr : 0) * rstride + col + k * 8;
    cp16(sm + r * (HD + 8) + k * 8, src, ok);
  }
}

using namespace spl::rngk;  // kG, kC, mix_post, keep_fast (rng_fast.cuh)

// 2^x, one MUFU.EX2 (flush-to-zero; the softmax operands are <= 0)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
struct Rng {
  uint64_t mixed;  // mix64(folded key)
  uint64_t tsh;    // thresh << 11
  bool on;         // p > 0
  __device__ explicit Rng(const DropKey& k) : mixed(k.mixed), tsh(k.thresh << 11), on(k.thresh != 0) {}
  __device__ __forceinline__ uint64_t row_base(uint64_t row_index, uint64_t s) const {
    return row_index * s + kC + kG;
  }
  __device__ __forceinline__ bool keep(uint64_t base, uint32_t key) const {
    if (!on) return true;
    return mix_post((mix_post(base + key) ^ mixed) + kG) >= tsh;
  }
};

// =====================================================================================
// softmax-dropout keep bits: bits[(hl*b + bj)*s + q][w] bit j = keep(q, 32w + j)
// The mask depends only on (seed, layer, op, microbatch) and the global {a,b,s,s} index, not
// on the data, so this RNG pass runs on a side stream concurrently with the tensor-core GEMMs
// that precede attention (it uses the ALU/FMA pipes the GEMM leaves idle).
// =====================================================================================
// One warp per (head, batch, query) row, lanes over the row's 32-key words. Within a word the
// high half of (row_base + key) and of the first xor-shift are loop-invariant (the carry out of
// the low half is checked once per word), so a key costs ~40 integer instructions.
// The hash is integer work split between the ALU pipe (LOP3/SHF/ISETP/IADD3) and the FMA-heavy
// pipe (IMAD*: the 64-bit constant multiplies). A 64-bit xor-shift can be 4 ALU ops (funnel
// shifts) or 2 ALU + 3 IMAD ops (multiplies by 2^(32-k)); with three shifts in IMAD form
// fmaheavy ran at 89% (ncu) and the all-funnel-shift form is 7% faster (tools/micro/
// bench_rng2.cu), so keep_fast uses funnel shifts throughout.

// The 32-key word (row base, keys kbeg..kbeg+31; bits at or past s cleared) of one query row.
template <bool TIE>
__device__ __forceinline__ uint32_t keep_word(const Rng& rng, uint64_t base, int kbeg, int s,
                                              uint32_t mixed_lo, uint32_t mixed_hi, uint32_t t_lo,
                                              uint32_t t_hi, const ShiftMuls& sm) {
  uint32_t word = 0;
  const uint64_t bw = base + (uint64_t)kbeg;
  const uint32_t blo = (uint32_t)bw, bhi = (uint32_t)(bw >> 32);
  const int kend = kbeg + 32 <= s ? 32 : s - kbeg;
  if (blo <= 0xffffffffu - 31u) {  // no carry into the high half inside this word
    const uint32_t hx = bhi ^ (bhi >> 30);
    const uint32_t hc = hx * 0x1ce4e5b9u;
    if ((blo >> 30) == ((blo + 31u) >> 30)) {
      const uint32_t c30 = __funnelshift_r(blo, bhi, 30);
      if constexpr (TIE) {
        // keep = hf > t_hi unless hf == t_hi (then the low word decides). hf = raw ^ (raw >> 31)
        // differs from raw in bit 0 only, so raw > t_hi decides too unless raw and t_hi agree
        // above bit 0 (raw - (t_hi & ~1) < 2, one IMAD + one compare instead of a shift, an xor
        // and a compare); such a key (2^-31) sends the word to the exact path below.
        bool tie = false;
        const uint32_t t_even = t_hi & ~1u;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t raw = hash_hi<true, true>(blo + j, bhi, hc, mixed_lo, mixed_hi, sm, c30);
          if (raw > t_hi) word |= 1u << j;
          tie |= raw - t_even < 2u;
        }
        if (tie) {  // a key near the threshold: decide every key of the word exactly
          word = 0;
#pragma unroll 1
          for (int j = 0; j < 32; ++j)
            if (keep_fast<true>(blo + j, bhi, hc, hx, mixed_lo, mixed_hi, t_lo, t_hi, sm, c30))
              word |= 1u << j;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (keep_fast<true>(blo + j, bhi, hc, hx, mixed_lo, mixed_hi, t_lo, t_hi, sm, c30))
            word |= 1u << j;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (keep_fast(blo + j, bhi, hc, hx, mixed_lo, mixed_hi, t_lo, t_hi, sm)) word |= 1u << j;
    }
  } else {
#pragma unroll 1
    for (int j = 0; j < 32; ++j) word |= (rng.keep(base, (uint32_t)(kbeg + j)) ? 1u : 0u) << j;
  }
  if (kend < 32) word &= (1u << kend) - 1u;
  return word;
}

template <bool TIE>
__global__ void __launch_bounds__(1024, 1) keep_bits_k(DropKey key, int64_t head_offset, int lh,
                                                   int b, int s, int W, int causal,
                                                   uint32_t* __restrict__ bits, ShiftMuls sm) {
  const Rng rng(key);
  const uint32_t mixed_lo = (uint32_t)rng.mixed, mixed_hi = (uint32_t)(rng.mixed >> 32);
  const uint32_t t_lo = (uint32_t)rng.tsh, t_hi = (uint32_t)(rng.tsh >> 32);
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int nrows = lh * b * s;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < nrows; row += warps) {
    const int q = row % s;
    const int t = row / s;
    const int bj = t % b, hl = t / b;
    const uint64_t base = rng.row_base(((uint64_t)(head_offset + hl) * b + bj) * s + q, s);
    uint32_t* out = bits + (int64_t)row * W;
    for (int w = lane; w < W; w += 32) {
      const int kbeg = 32 * w;
      out[w] = (causal && kbeg > q)
                   ? 0u
                   : keep_word<TIE>(rng, base, kbeg, s, mixed_lo, mixed_hi, t_lo, t_hi, sm);
    }
  }
}

// Transposed layout for the fused backward (thread = key): bits[((hl*b + bj)*(s/32) + qb)*s + k]
// bit j = keep(32*qb + j, k). One warp per 32 query rows (lane = row, so every lane hashes its
// own row's words exactly as keep_bits_k does), each 32 x 32 block transposed across the warp
// and stored coalesced (lanes = consecutive keys). s % 32 == 0.
__device__ __forceinline__ uint32_t warp_transpose32_k(uint32_t x, int lane) {
  uint32_t m = 0x0000ffffu;
#pragma unroll
  for (int j = 16; j != 0; j >>= 1, m ^= m << j) {
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y & m) << j));
  }
  return x;
}
template <bool TIE>
__global__ void __launch_bounds__(1024, 1) keep_bits_t_k(DropKey key, int64_t head_offset, int lh,
                                                     int b, int s, int causal,
                                                     uint32_t* __restrict__ bits, ShiftMuls sm) {
  const Rng rng(key);
  const uint32_t mixed_lo = (uint32_t)rng.mixed, mixed_hi = (uint32_t)(rng.mixed >> 32);
  const uint32_t t_lo = (uint32_t)rng.tsh, t_hi = (uint32_t)(rng.tsh >> 32);
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int nqb = s / 32, W = s / 32;
  const int nunits = lh * b * nqb * W;  // (32-row block, key word): fine-grained for balance
  for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nunits; u += warps) {
    const int w = u % W;
    const int blk = u / W;
    const int qb = blk % nqb;
    const int t = blk / nqb;
    const int bj = t % b, hl = t / b;
    uint32_t word = 0;
    if (!causal || w <= qb) {  // key words past the block's last query: all masked
      const int q = 32 * qb + lane;
      const uint64_t base = rng.row_base(((uint64_t)(head_offset + hl) * b + bj) * s + q, s);
      word = keep_word<TIE>(rng, base, 32 * w, s, mixed_lo, mixed_hi, t_lo, t_hi, sm);
      word = warp_transpose32_k(word, lane);
    }
    bits[(int64_t)blk * s + 32 * w + lane] = word;
  }
}

// =====================================================================================
// forward
// =====================================================================================
template <int HD, bool CAUSAL, bool MAT>
__global__ void __launch_bounds__(128) fa_fwd(AttnArgs a) {
  constexpr int BM = 64, BN = 64, LDS = HD + 8, NT = 128;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* Qs = reinterpret_cast<bf16*>(smem_raw);
  bf16* Ks = Qs + BM * LDS;      // [2][BN][LDS]
  bf16* Vs = Ks + 2 * BN * LDS;  // [2][BN][LDS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int q0 = blockIdx.x * BM;
  const int hl = blockIdx.y / (int)a.b, bj = blockIdx.y % (int)a.b;
  const int S = (int)a.s;
  const bf16* base = static_cast<const bf16*>(a.qkv) + (int64_t)bj * a.ld;
  const int64_t rstride = a.b * a.ld;
  const int64_t qcol = a.qoff + (int64_t)hl * HD, kcol = a.koff + (int64_t)hl * HD,
                vcol = a.voff + (int64_t)hl * HD;
  const bool drop_on = a.drop.thresh != 0;
  const int W = (S + 31) / 32;
  const int64_t brow = ((int64_t)hl * a.b + bj) * a.s;  // keep-bit / lse row base
  // MAT (materialised interior, causal included) visits every key tile; otherwise causal
  // stops at the diagonal.
  const int kv_end = (CAUSAL && !MAT) ? min(S, q0 + BM) : S;
  const int nkv = (kv_end + BN - 1) / BN;
  const int row0 = q0 + warp * 16 + g;  // this thread's rows: row0, row0 + 8
  const float sl2 = a.scale * kLog2e;

  uint32_t qf[HD / 16][4];
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};

  auto scores = [&](const bf16* Kb, float (&sacc)[BN / 8][4], int k0) {
#pragma unroll
    for (int i = 0; i < BN / 8; ++i) sacc[i][0] = sacc[i][1] = sacc[i][2] = sacc[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int nb = 0; nb < BN / 8; nb += 2) {
        uint32_t b[4];
        ldsm_x4(b, Kb + (nb * 8 + (lane & 7) + (lane >> 4) * 8) * LDS + kk * 16 + ((lane >> 3) & 1) * 8);
        mma16816(sacc[nb], qf[kk], b[0], b[1]);
        mma16816(sacc[nb + 1], qf[kk], b[2], b[3]);
      }
    }
    const bool edge = (k0 + BN > S) || (CAUSAL && k0 + BN - 1 > q0 + warp * 16);
#pragma unroll
    for (int nb = 0; nb < BN / 8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = sacc[nb][e] * sl2;
        if (edge) {
          const int key = k0 + nb * 8 + 2 * tq + (e & 1);
          const int qr = row0 + (e >> 1) * 8;
          if (key >= S || (CAUSAL && key > qr)) v = -INFINITY;
        }
        sacc[nb][e] = v;
      }
  };

  load_tile<HD, BM, NT>(Qs, base, q0, a.s, rstride, qcol);
  if (MAT) {
    // ---- pass 1: exact row max and sum (K tiles only)
    load_tile<HD, BN, NT>(Ks, base, 0, a.s, rstride, kcol);
    cp_commit();
    for (int jb = 0; jb < nkv; ++jb) {
      const int buf = jb & 1;
      if (jb + 1 < nkv) {
        load_tile<HD, BN, NT>(Ks + (buf ^ 1) * BN * LDS, base, (int64_t)(jb + 1) * BN, a.s, rstride, kcol);
        cp_commit();
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      if (jb == 0) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ldsm_x4(qf[kk], Qs + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
      }
      float sacc[BN / 8][4];
      scores(Ks + buf * BN * LDS, sacc, jb * BN);
      float mx[2] = {m[0], m[1]};
#pragma unroll
      for (int nb = 0; nb < BN / 8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) mx[e >> 1] = fmaxf(mx[e >> 1], sacc[nb][e]);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
        l[r] *= (m[r] == -INFINITY) ? 0.f : ex2(m[r] - mx[r]);
        m[r] = mx[r];
      }
#pragma unroll
      for (int nb = 0; nb < BN / 8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float mr = m[e >> 1] == -INFINITY ? 0.f : m[e >> 1];
          l[e >> 1] += ex2(sacc[nb][e] - mr);
        }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
      l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
    }
  }
  load_tile<HD, BN, NT>(Ks, base, 0, a.s, rstride, kcol);
  load_tile<HD, BN, NT>(Vs, base, 0, a.s, rstride, vcol);
  cp_commit();
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  const float inv_l[2] = {MAT ? 1.f / l[0] : 1.f, MAT ? 1.f / l[1] : 1.f};

  for (int jb = 0; jb < nkv; ++jb) {
    const int buf = jb & 1;
    if (jb + 1 < nkv) {
      load_tile<HD, BN, NT>(Ks + (buf ^ 1) * BN * LDS, base, (int64_t)(jb + 1) * BN, a.s, rstride, kcol);
      load_tile<HD, BN, NT>(Vs + (buf ^ 1) * BN * LDS, base, (int64_t)(jb + 1) * BN, a.s, rstride, vcol);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (!MAT && jb == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(qf[kk], Qs + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
    }
    const int k0 = jb * BN;
    float sacc[BN / 8][4];
    scores(Ks + buf * BN * LDS, sacc, k0);
    if (!MAT) {
      float mx[2] = {m[0], m[1]};
#pragma unroll
      for (int nb = 0; nb < BN / 8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) mx[e >> 1] = fmaxf(mx[e >> 1], sacc[nb][e]);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
        const float corr = (m[r] == -INFINITY) ? 0.f : ex2(m[r] - mx[r]);
        m[r] = mx[r];
        l[r] *= corr;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
          o[i][2 * r] *= corr;
          o[i][2 * r + 1] *= corr;
        }
      }
    }
    const float mr[2] = {m[0] == -INFINITY ? 0.f : m[0], m[1] == -INFINITY ? 0.f : m[1]};
    uint32_t kw[2][2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const int qr = row0 + r * 8, wd = k0 / 32 + w;
        kw[r][w] = !drop_on ? 0xffffffffu : (qr < S && wd < W) ? a.keepbits[(brow + qr) * W + wd] : 0u;
      }
    uint32_t pa[BN / 16][4];
#pragma unroll
    for (int nb = 0; nb < BN / 8; ++nb) {
      float p[4], pd[4];
      bool kp[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        float pv = ex2(sacc[nb][e] - mr[r]);
        if (!MAT) l[r] += pv;
        else pv *= inv_l[r];
        const int kl = nb * 8 + 2 * tq + (e & 1);
        const bool bit = (kw[r][kl >> 5] >> (kl & 31)) & 1u;
        kp[e] = bit && (MAT ? k0 + kl < S : pv != 0.f);
        p[e] = pv;
        pd[e] = kp[e] ? pv * a.drop.inv_keep : 0.f;
      }
      if (MAT) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int qr = row0 + r * 8;
          const int key = k0 + nb * 8 + 2 * tq;
          if (qr < S && key < S) {  // S even in MAT mode (checked by the dispatcher)
            const int64_t mi = (((int64_t)hl * a.b + bj) * a.s + qr) * a.s + key;
            *reinterpret_cast<uint32_t*>(static_cast<bf16*>(a.sm) + mi) = pack_bf16(p[2 * r], p[2 * r + 1]);
            *reinterpret_cast<uint32_t*>(static_cast<bf16*>(a.sd) + mi) = pack_bf16(pd[2 * r], pd[2 * r + 1]);
            *reinterpret_cast<uint16_t*>(a.mask + mi) =
                (uint16_t)((kp[2 * r] ? 1 : 0) | ((kp[2 * r + 1] ? 1 : 0) << 8));
          }
        }
      }
      const int kk2 = nb >> 1, hi = nb & 1;
      pa[kk2][hi * 2 + 0] = pack_bf16(pd[0], pd[1]);
      pa[kk2][hi * 2 + 1] = pack_bf16(pd[2], pd[3]);
    }
    const bf16* Vb = Vs + buf * BN * LDS;
#pragma unroll
    for (int kk2 = 0; kk2 < BN / 16; ++kk2) {
#pragma unroll
      for (int db = 0; db < HD / 8; db += 2) {
        uint32_t b[4];
        ldsm_x4_t(b, Vb + (kk2 * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + db * 8 + (lane >> 4) * 8);
        mma16816(o[db], pa[kk2], b[0], b[1]);
        mma16816(o[db + 1], pa[kk2], b[2], b[3]);
      }
    }
    __syncthreads();
  }
  if (!MAT) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
      l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
    }
  }
  bf16* out = static_cast<bf16*>(a.o);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qr = row0 + r * 8;
    if (qr >= S) continue;
    const float inv = MAT ? 1.f : 1.f / l[r];
    bf16* orow = out + ((int64_t)qr * a.b + bj) * a.ldo + (int64_t)hl * HD;
#pragma unroll
    for (int db = 0; db < HD / 8; ++db)
      *reinterpret_cast<uint32_t*>(orow + db * 8 + 2 * tq) =
          pack_bf16(o[db][2 * r] * inv, o[db][2 * r + 1] * inv);
    if (tq == 0 && a.lse) a.lse[brow + qr] = (m[r] + log2f(l[r])) * kLn2;
  }
}

// =====================================================================================
// backward: delta = rowsum(dO ∘ O)
// =====================================================================================
template <int HD>
__global__ void fa_delta(AttnArgs a, const bf16* __restrict__ dout, float* __restrict__ delta) {
  // rowdot_i = dO_i·O_i of every (head, batch, query) row. Rows are visited in memory order
  // (token-major, heads of one token contiguous), 4 lanes per row with interleaved 16-byte
  // vectors, so a warp streams 8 consecutive rows = one contiguous span of dO and of O.
  static_assert(HD % 32 == 0, "fa_delta: head_dim must be a multiple of 32");
  constexpr int VPL = HD / 32;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = t >> 2;
  const int sub = (int)(t & 3);
  const int64_t nrows = a.lh * a.b * a.s;
  const int64_t hl = r % a.lh, tok = r / a.lh;  // tok = i*b + bj
  const bf16* o = static_cast<const bf16*>(a.o);
  float acc = 0.f;
  if (r < nrows) {
    const int64_t off = tok * a.ldo + hl * HD;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int c = (sub + 4 * v) * 8;
      const uint4 x = *reinterpret_cast<const uint4*>(dout + off + c);
      const uint4 y = *reinterpret_cast<const uint4*>(o + off + c);
      const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        acc += __uint_as_float(xs[k] << 16) * __uint_as_float(ys[k] << 16) +
               __uint_as_float(xs[k] & 0xffff0000u) * __uint_as_float(ys[k] & 0xffff0000u);
    }
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  if (sub == 0 && r < nrows) {
    const int64_t bj = tok % a.b, i = tok / a.b;
    delta[(hl * a.b + bj) * a.s + i] = acc;
  }
}

// =====================================================================================
// backward: dK, dV (key-parallel). Recompute regimes also emit the keep bits for fa_bwd_dq.
// =====================================================================================
template <int HD, bool CAUSAL, bool STORED>
__global__ void __launch_bounds__(128) fa_bwd_dkdv(AttnArgs a, const bf16* __restrict__ dout,
                                                   bf16* __restrict__ dqkv,
                                                   const float* __restrict__ delta) {
  constexpr int BK_ = 64, BQ = 32, LDS = HD + 8, NT = 128;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* Ks = reinterpret_cast<bf16*>(smem_raw);
  bf16* Vs = Ks + BK_ * LDS;
  bf16* Qs = Vs + BK_ * LDS;       // [2][BQ][LDS]
  bf16* Ds = Qs + 2 * BQ * LDS;    // [2][BQ][LDS] dO
  float* lse_s = reinterpret_cast<float*>(Ds + 2 * BQ * LDS);  // [2][BQ]
  float* dl_s = lse_s + 2 * BQ;                                // [2][BQ]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int k0 = blockIdx.x * BK_;
  const int hl = blockIdx.y / (int)a.b, bj = blockIdx.y % (int)a.b;
  const int S = (int)a.s;
  const bf16* base = static_cast<const bf16*>(a.qkv) + (int64_t)bj * a.ld;
  const bf16* dbase = dout + (int64_t)bj * a.ldo;
  const int64_t rstride = a.b * a.ld, dstride = a.b * a.ldo;
  const int64_t qcol = a.qoff + (int64_t)hl * HD, kcol = a.koff + (int64_t)hl * HD,
                vcol = a.voff + (int64_t)hl * HD;
  const int64_t rowbase = ((int64_t)hl * a.b + bj) * a.s;  // lse/delta/bits row index base
  const float sl2 = a.scale * kLog2e;
  const bool drop_on = a.drop.thresh != 0;
  const int W = (S + 31) / 32;
  const int kword = k0 / 32 + warp / 2;          // the 32-key word holding this warp's keys
  const int kbit = (warp & 1) * 16 + g;          // bit of key0 in that word (key0 + 8: +8)

  const int q_start = CAUSAL ? (k0 / BQ) * BQ : 0;
  const int nq = (S - q_start + BQ - 1) / BQ;

  auto load_q = [&](int it, int buf) {
    const int qb = q_start + it * BQ;
    load_tile<HD, BQ, NT>(Qs + buf * BQ * LDS, base, qb, a.s, rstride, qcol);
    load_tile<HD, BQ, NT>(Ds + buf * BQ * LDS, dbase, qb, a.s, dstride, (int64_t)hl * HD);
    if (threadIdx.x < BQ) {
      const int q = qb + threadIdx.x;
      lse_s[buf * BQ + threadIdx.x] = (q < S && !STORED) ? a.lse[rowbase + q] * kLog2e : INFINITY;
      dl_s[buf * BQ + threadIdx.x] = q < S ? delta[rowbase + q] : 0.f;
    }
  };
  load_tile<HD, BK_, NT>(Ks, base, k0, a.s, rstride, kcol);
  load_tile<HD, BK_, NT>(Vs, base, k0, a.s, rstride, vcol);
  load_q(0, 0);
  cp_commit();

  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int key0 = k0 + warp * 16 + g;  // rows of this thread: key0, key0 + 8

  for (int it = 0; it < nq; ++it) {
    const int buf = it & 1;
    __syncthreads();  // all warps done with iteration it-1
    if (it + 1 < nq) {
      load_q(it + 1, buf ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const bf16* Qb = Qs + buf * BQ * LDS;
    const bf16* Db = Ds + buf * BQ * LDS;
    const float* lq = lse_s + buf * BQ;
    const float* dq_ = dl_s + buf * BQ;
    const int qb = q_start + it * BQ;
    float st[BQ / 8][4], dpt[BQ / 8][4];
#pragma unroll
    for (int i = 0; i < BQ / 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[i][e] = dpt[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t ka[4], va[4];
      ldsm_x4(ka, Ks + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
      ldsm_x4(va, Vs + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
#pragma unroll
      for (int nb = 0; nb < BQ / 8; nb += 2) {
        uint32_t b[4], c[4];
        ldsm_x4(b, Qb + (nb * 8 + (lane & 7) + (lane >> 4) * 8) * LDS + kk * 16 + ((lane >> 3) & 1) * 8);
        mma16816(st[nb], ka, b[0], b[1]);
        mma16816(st[nb + 1], ka, b[2], b[3]);
        ldsm_x4(c, Db + (nb * 8 + (lane & 7) + (lane >> 4) * 8) * LDS + kk * 16 + ((lane >> 3) & 1) * 8);
        mma16816(dpt[nb], va, c[0], c[1]);
        mma16816(dpt[nb + 1], va, c[2], c[3]);
      }
    }
    const bool edge = (qb + BQ > S) || (k0 + BK_ > S) || (CAUSAL && qb < k0 + warp * 16 + 16);
    uint32_t pa[BQ / 16][4], da[BQ / 16][4];
#pragma unroll
    for (int nb = 0; nb < BQ / 8; ++nb) {
      float pd[4], ds[4];
#pragma unroll
      for (int par = 0; par < 2; ++par) {
        const int qi = nb * 8 + 2 * tq + par;
        const int q = qb + qi;
        const float lqv = lq[qi], dqv = dq_[qi];
        const uint32_t kwd = (STORED || !drop_on) ? 0xffffffffu
                             : (q < S && kword < W) ? a.keepbits[(rowbase + q) * W + kword] : 0u;
#pragma unroll
        for (int kr = 0; kr < 2; ++kr) {
          const int e = kr * 2 + par;
          const int key = key0 + kr * 8;
          const bool valid = !edge || (q < S && key < S && !(CAUSAL && key > q));
          float p = 0.f, pdv = 0.f;
          bool keep = false;
          if (STORED) {
            if (valid) {
              const int64_t mi = (rowbase + q) * a.s + key;
              p = __bfloat162float(static_cast<const bf16*>(a.sm)[mi]);
              keep = a.mask[mi] != 0;
              pdv = __bfloat162float(static_cast<const bf16*>(a.sd)[mi]);
            }
          } else {
            p = valid ? ex2(st[nb][e] * sl2 - lqv) : 0.f;
            keep = ((kwd >> (kbit + kr * 8)) & 1u) && p != 0.f;
            pdv = keep ? p * a.drop.inv_keep : 0.f;
          }
          pd[e] = pdv;
          const float dp = keep ? dpt[nb][e] * a.drop.inv_keep : 0.f;
          ds[e] = p * (dp - dqv);
        }
      }
      const int kk2 = nb >> 1, hi = nb & 1;
      pa[kk2][hi * 2 + 0] = pack_bf16(pd[0], pd[1]);
      pa[kk2][hi * 2 + 1] = pack_bf16(pd[2], pd[3]);
      da[kk2][hi * 2 + 0] = pack_bf16(ds[0], ds[1]);
      da[kk2][hi * 2 + 1] = pack_bf16(ds[2], ds[3]);
    }
#pragma unroll
    for (int kk2 = 0; kk2 < BQ / 16; ++kk2) {
#pragma unroll
      for (int db = 0; db < HD / 8; db += 2) {
        uint32_t b[4], c[4];
        ldsm_x4_t(b, Db + (kk2 * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + db * 8 + (lane >> 4) * 8);
        mma16816(dv[db], pa[kk2], b[0], b[1]);
        mma16816(dv[db + 1], pa[kk2], b[2], b[3]);
        ldsm_x4_t(c, Qb + (kk2 * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + db * 8 + (lane >> 4) * 8);
        mma16816(dk[db], da[kk2], c[0], c[1]);
        mma16816(dk[db + 1], da[kk2], c[2], c[3]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = key0 + r * 8;
    if (key >= S) continue;
    bf16* row = dqkv + ((int64_t)key * a.b + bj) * a.ld;
#pragma unroll
    for (int db = 0; db < HD / 8; ++db) {
      *reinterpret_cast<uint32_t*>(row + kcol + db * 8 + 2 * tq) =
          pack_bf16(dk[db][2 * r] * a.scale, dk[db][2 * r + 1] * a.scale);
      *reinterpret_cast<uint32_t*>(row + vcol + db * 8 + 2 * tq) =
          pack_bf16(dv[db][2 * r], dv[db][2 * r + 1]);
    }
  }
}

// =====================================================================================
// backward: dQ (query-parallel); keep bits from fa_bwd_dkdv (or the stored mask)
// =====================================================================================
template <int HD, bool CAUSAL, bool STORED>
__global__ void __launch_bounds__(128) fa_bwd_dq(AttnArgs a, const bf16* __restrict__ dout,
                                                 bf16* __restrict__ dqkv,
                                                 const float* __restrict__ delta) {
  constexpr int BM = 64, BN = 32, LDS = HD + 8, NT = 128;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* Qs = reinterpret_cast<bf16*>(smem_raw);
  bf16* Ds = Qs + BM * LDS;
  bf16* Ks = Ds + BM * LDS;       // [2][BN][LDS]
  bf16* Vs = Ks + 2 * BN * LDS;   // [2][BN][LDS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int q0 = blockIdx.x * BM;
  const int hl = blockIdx.y / (int)a.b, bj = blockIdx.y % (int)a.b;
  const int S = (int)a.s;
  const bf16* base = static_cast<const bf16*>(a.qkv) + (int64_t)bj * a.ld;
  const bf16* dbase = dout + (int64_t)bj * a.ldo;
  const int64_t rstride = a.b * a.ld, dstride = a.b * a.ldo;
  const int64_t qcol = a.qoff + (int64_t)hl * HD, kcol = a.koff + (int64_t)hl * HD,
                vcol = a.voff + (int64_t)hl * HD;
  const int64_t rowbase = ((int64_t)hl * a.b + bj) * a.s;
  const float sl2 = a.scale * kLog2e;
  const int kv_end = CAUSAL ? min(S, q0 + BM) : S;
  const int nkv = (kv_end + BN - 1) / BN;
  const int W = (S + 31) / 32;
  const bool bits_on = a.drop.thresh != 0;

  load_tile<HD, BM, NT>(Qs, base, q0, a.s, rstride, qcol);
  load_tile<HD, BM, NT>(Ds, dbase, q0, a.s, dstride, (int64_t)hl * HD);
  load_tile<HD, BN, NT>(Ks, base, 0, a.s, rstride, kcol);
  load_tile<HD, BN, NT>(Vs, base, 0, a.s, rstride, vcol);
  cp_commit();

  const int row0 = q0 + warp * 16 + g;
  float lse[2], dl[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = row0 + r * 8;
    lse[r] = (q < S && !STORED) ? a.lse[rowbase + q] * kLog2e : INFINITY;
    dl[r] = q < S ? delta[rowbase + q] : 0.f;
  }
  uint32_t qf[HD / 16][4], df[HD / 16][4];
  float dq[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int jb = 0; jb < nkv; ++jb) {
    const int buf = jb & 1;
    if (jb + 1 < nkv) {
      load_tile<HD, BN, NT>(Ks + (buf ^ 1) * BN * LDS, base, (int64_t)(jb + 1) * BN, a.s, rstride, kcol);
      load_tile<HD, BN, NT>(Vs + (buf ^ 1) * BN * LDS, base, (int64_t)(jb + 1) * BN, a.s, rstride, vcol);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (jb == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        ldsm_x4(qf[kk], Qs + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
        ldsm_x4(df[kk], Ds + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
      }
    }
    const int kb0 = jb * BN;
    uint32_t word[2] = {0xffffffffu, 0xffffffffu};
    if (!STORED && bits_on) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int q = row0 + r * 8;
        word[r] = q < S ? a.keepbits[(rowbase + q) * W + kb0 / 32] : 0u;
      }
    }
    const bf16* Kb = Ks + buf * BN * LDS;
    const bf16* Vb = Vs + buf * BN * LDS;
    float sc[BN / 8][4], dp[BN / 8][4];
#pragma unroll
    for (int i = 0; i < BN / 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[i][e] = dp[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int nb = 0; nb < BN / 8; nb += 2) {
        uint32_t b[4], c[4];
        ldsm_x4(b, Kb + (nb * 8 + (lane & 7) + (lane >> 4) * 8) * LDS + kk * 16 + ((lane >> 3) & 1) * 8);
        mma16816(sc[nb], qf[kk], b[0], b[1]);
        mma16816(sc[nb + 1], qf[kk], b[2], b[3]);
        ldsm_x4(c, Vb + (nb * 8 + (lane & 7) + (lane >> 4) * 8) * LDS + kk * 16 + ((lane >> 3) & 1) * 8);
        mma16816(dp[nb], df[kk], c[0], c[1]);
        mma16816(dp[nb + 1], df[kk], c[2], c[3]);
      }
    }
    const bool edge = (kb0 + BN > S) || (q0 + BM > S) || (CAUSAL && kb0 + BN - 1 > q0 + warp * 16);
    uint32_t da[BN / 16][4];
#pragma unroll
    for (int nb = 0; nb < BN / 8; ++nb) {
      float ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const int kl = nb * 8 + 2 * tq + (e & 1);
        const int key = kb0 + kl;
        const int q = row0 + r * 8;
        const bool valid = !edge || (q < S && key < S && !(CAUSAL && key > q));
        float p = 0.f;
        bool keep = false;
        if (valid) {
          if (STORED) {
            const int64_t mi = (rowbase + q) * a.s + key;
            p = __bfloat162float(static_cast<const bf16*>(a.sm)[mi]);
            keep = a.mask[mi] != 0;
          } else {
            p = ex2(sc[nb][e] * sl2 - lse[r]);
            keep = (word[r] >> kl) & 1u;
          }
        }
        const float d = keep ? dp[nb][e] * a.drop.inv_keep : 0.f;
        ds[e] = p * (d - dl[r]);
      }
      const int kk2 = nb >> 1, hi = nb & 1;
      da[kk2][hi * 2 + 0] = pack_bf16(ds[0], ds[1]);
      da[kk2][hi * 2 + 1] = pack_bf16(ds[2], ds[3]);
    }
#pragma unroll
    for (int kk2 = 0; kk2 < BN / 16; ++kk2) {
#pragma unroll
      for (int db = 0; db < HD / 8; db += 2) {
        uint32_t b[4];
        ldsm_x4_t(b, Kb + (kk2 * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + db * 8 + (lane >> 4) * 8);
        mma16816(dq[db], da[kk2], b[0], b[1]);
        mma16816(dq[db + 1], da[kk2], b[2], b[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = row0 + r * 8;
    if (q >= S) continue;
    bf16* row = dqkv + ((int64_t)q * a.b + bj) * a.ld + qcol;
#pragma unroll
    for (int db = 0; db < HD / 8; ++db)
      *reinterpret_cast<uint32_t*>(row + db * 8 + 2 * tq) =
          pack_bf16(dq[db][2 * r] * a.scale, dq[db][2 * r + 1] * a.scale);
  }
}

template <int HD, bool CAUSAL, bool MAT>
void launch_fwd_t(const AttnArgs& a, cudaStream_t st) {
  constexpr int LDS = HD + 8;
  const int smem = (64 * LDS + 4 * 64 * LDS) * 2;
  static bool once = [&] {
    SPL_CUDA(cudaFuncSetAttribute(fa_fwd<HD, CAUSAL, MAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return true;
  }();
  (void)once;
  dim3 grid((unsigned)((a.s + 63) / 64), (unsigned)(a.lh * a.b));
  fa_fwd<HD, CAUSAL, MAT><<<grid, 128, smem, st>>>(a);
  SPL_CHECK_LAUNCH();
}

template <int HD, bool CAUSAL, bool STORED>
void launch_bwd_t(const AttnArgs& a, const bf16* dout, bf16* dqkv, float* delta, cudaStream_t st) {
  constexpr int LDS = HD + 8;
  const int64_t rows = a.lh * a.b * a.s;
  fa_delta<HD><<<(unsigned)((rows * 4 + 255) / 256), 256, 0, st>>>(a, dout, delta);
  SPL_CHECK_LAUNCH();
  const int smem_kv = (2 * 64 * LDS + 4 * 32 * LDS) * 2 + 4 * 32 * 4;
  const int smem_q = (2 * 64 * LDS + 4 * 32 * LDS) * 2;
  static bool once = [&] {
    SPL_CUDA(cudaFuncSetAttribute(fa_bwd_dkdv<HD, CAUSAL, STORED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv));
    SPL_CUDA(cudaFuncSetAttribute(fa_bwd_dq<HD, CAUSAL, STORED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q));
    return true;
  }();
  (void)once;
  dim3 grid((unsigned)((a.s + 63) / 64), (unsigned)(a.lh * a.b));
  fa_bwd_dkdv<HD, CAUSAL, STORED><<<grid, 128, smem_kv, st>>>(a, dout, dqkv, delta);
  SPL_CHECK_LAUNCH();
  fa_bwd_dq<HD, CAUSAL, STORED><<<grid, 128, smem_q, st>>>(a, dout, dqkv, delta);
  SPL_CHECK_LAUNCH();
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

template <typename T>
bool attn_tc_supported(const AttnArgs& a);
template <typename T>
void attn_fwd_tc(const AttnArgs& a, cudaStream_t st);
template <typename T>
void attn_bwd_tc(const AttnArgs& a, const void* dout, void* dqkv, float* delta, cudaStream_t st);

template <>
bool attn_tc_supported<bf16>(const AttnArgs& a) {
  const bool hd_ok = a.hd == 32 || a.hd == 64 || a.hd == 96 || a.hd == 128 || a.hd == 160;
  const bool mat = a.sm != nullptr;
  return hd_ok && a.ld % 8 == 0 && a.ldo % 8 == 0 && a.qoff % 8 == 0 && a.koff % 8 == 0 &&
         a.voff % 8 == 0 && aligned16(a.qkv) && aligned16(a.o) && a.s < (1 << 30) &&
         (mat ? (a.s % 2 == 0 && a.mask != nullptr && a.sd != nullptr) : a.lse != nullptr);
}

#define SPL_HD_SWITCH(HDV, ...)                                   \
  switch (HDV) {                                                   \
    case 32: { constexpr int HD = 32; __VA_ARGS__; break; }       \
    case 64: { constexpr int HD = 64; __VA_ARGS__; break; }       \
    case 96: { constexpr int HD = 96; __VA_ARGS__; break; }       \
    case 128: { constexpr int HD = 128; __VA_ARGS__; break; }     \
    case 160: { constexpr int HD = 160; __VA_ARGS__; break; }     \
    default: raise(3, "attention: unsupported head_dim");          \
  }

template <>
void attn_fwd_tc<bf16>(const AttnArgs& a, cudaStream_t st) {
  require(a.keepbits != nullptr || a.drop.thresh == 0, "attention forward: keep-bit buffer missing");
  static const bool umma_off = [] {
    const char* e = std::getenv("SPL_ATTN_UMMA");
    return e != nullptr && e[0] == '0';
  }();
  if (!umma_off && attn_fwd_umma_supported(a)) {
    attn_fwd_umma(a, st);
    return;
  }
  const bool mat = a.sm != nullptr;
  SPL_HD_SWITCH(a.hd, {
    if (a.causal) {
      if (mat) launch_fwd_t<HD, true, true>(a, st); else launch_fwd_t<HD, true, false>(a, st);
    } else {
      if (mat) launch_fwd_t<HD, false, true>(a, st); else launch_fwd_t<HD, false, false>(a, st);
    }
  });
}

static bool umma_bwd_on(const AttnArgs& a) {
  static const bool off = [] {
    const char* e = std::getenv("SPL_ATTN_UMMA");
    return e != nullptr && e[0] == '0';
  }();
  return !off && attn_bwd_umma_supported(a);
}

bool attn_bwd_uses_fused(const AttnArgs& a) { return umma_bwd_on(a) && attn_bwd_fused_supported(a); }

template <>
void attn_bwd_tc<bf16>(const AttnArgs& a, const void* dout, void* dqkv, float* delta,
                       cudaStream_t st) {
  const bool stored = a.sm != nullptr;
  if (attn_bwd_uses_fused(a)) {
    attn_bwd_fused(a, dout, dqkv, st);
    return;
  }
  require(!a.keep_t, "attention backward: transposed keep bits need the fused path");
  if (umma_bwd_on(a)) {  // recompute regimes and (stored interior) the no-recompute regime
    const int64_t rows = a.lh * a.b * a.s;
    SPL_HD_SWITCH(a.hd, fa_delta<HD><<<(unsigned)((rows * 4 + 255) / 256), 256, 0, st>>>(
                            a, static_cast<const bf16*>(dout), delta));
    SPL_CHECK_LAUNCH();
    attn_bwd_umma(a, dout, dqkv, delta, st);
    return;
  }
  if (!stored) require(a.keepbits != nullptr || a.drop.thresh == 0, "attention backward: keep-bit buffer missing");
  const bf16* d = static_cast<const bf16*>(dout);
  bf16* g = static_cast<bf16*>(dqkv);
  SPL_HD_SWITCH(a.hd, {
    if (a.causal) {
      if (stored) launch_bwd_t<HD, true, true>(a, d, g, delta, st); else launch_bwd_t<HD, true, false>(a, d, g, delta, st);
    } else {
      if (stored) launch_bwd_t<HD, false, true>(a, d, g, delta, st); else launch_bwd_t<HD, false, false>(a, d, g, delta, st);
    }
  });
}

void attn_keep_bits(const AttnArgs& a, cudaStream_t st) {
  if (a.drop.thresh == 0 || a.keepbits == nullptr) return;
  require(a.lh * a.b * a.s < (1ll << 31), "keep bits: too many rows");
  const int W = (int)((a.s + 31) / 32);
  const int64_t rows = a.lh * a.b * a.s;
  // one 1024-thread CTA per SM (64 registers a thread: more independent hashes in flight per
  // warp than 8 x 256 threads at 32 registers; 1.84 vs 1.92 ms per 22B pass, bench_rng2.cu)
  int64_t grid = (rows + 31) / 32;  // 32 warps (rows) per CTA
  if (grid > kNumSMs) grid = kNumSMs;
  static const bool tie = [] {
    const char* e = std::getenv("SPL_RNG_TIE");
    return !(e != nullptr && e[0] == '0');
  }();
  auto kern = tie ? keep_bits_k<true> : keep_bits_k<false>;
  // causal: words above the diagonal are skipped (their probabilities are 0), except when the
  // interior is materialised — the stored mask carries the raw keep bit at every position,
  // masked or not (mask_slice, block.cpp:392-394)
  const int causal_skip = a.causal && a.sm == nullptr;
  if (a.keep_t) {  // the fused backward's (key, 32 queries) words
    require(a.s % 32 == 0, "keep bits (transposed): s % 32 != 0");
    require(rows / 32 * W < (1ll << 31), "keep bits (transposed): too many words");
    int64_t gt = (rows / 32 * W + 31) / 32;
    if (gt > kNumSMs) gt = kNumSMs;
    auto kt = tie ? keep_bits_t_k<true> : keep_bits_t_k<false>;
    kt<<<(unsigned)gt, 1024, 0, st>>>(a.drop, a.head_offset, (int)a.lh, (int)a.b, (int)a.s,
                                      causal_skip, a.keepbits, ShiftMuls{4u, 32u, 2u, 1u});
    SPL_CHECK_LAUNCH();
    return;
  }
  kern<<<(unsigned)grid, 1024, 0, st>>>(a.drop, a.head_offset, (int)a.lh, (int)a.b, (int)a.s, W,
                                        causal_skip, a.keepbits, ShiftMuls{4u, 32u, 2u, 1u});
  SPL_CHECK_LAUNCH();
}

}  // namespace spl::k
