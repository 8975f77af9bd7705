// Attention backward on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), bf16, for the
// recompute regimes (selective / full): nothing of the s×s interior comes from HBM.
//
// fa_bwd_dkdv_umma — CTA = 128 keys of one (head, batch), loops over 64-query tiles:
//   MMA   Sᵀ = K·Qᵀ, dPᵀ = V·dOᵀ  (M=128 keys, N=64 queries)          -> TMEM (2 buffers)
//   warps Pᵀ = exp2(Sᵀc - lse), keep from the keep-bit buffer (attn_keep_bits: one word per
//         (query, 32 keys) = one warp's keys, broadcast by shuffle),
//         P̃ᵀ = Pᵀ·keep/(1-p), dSᵀ = Pᵀ∘(dPᵀ·keep/(1-p) - rowdot)   -> bf16 smem (UMMA layout)
//   MMA   dV += P̃ᵀ·dO, dK += dSᵀ·Q  (M=128, N=HD, K=64)               -> TMEM
// fa_bwd_dq_umma — CTA = 128 queries, loops over 64-key tiles:
//   MMA   S = Q·Kᵀ, dP = dO·Vᵀ; warps dS (same keep bits); MMA dQ += dS·K.
// The counter-RNG pass that fills the keep bits (attn_keep_bits) runs once per backward.
#include <cstring>
#include <type_traits>
#include <mutex>
#include <unordered_map>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace spl::k {

CUtensorMap attn_seq_map(const void* ptr, int64_t width, int64_t b, int64_t s, int64_t ld, int rows);
using EncodeFnB = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFnB encode_fn_bwd() {
  static EncodeFnB fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    SPL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (p == nullptr || q != cudaDriverEntryPointSuccess) raise(3, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFnB>(p);
  }();
  return fn;
}

// L2 prefetch of a TMA box (no shared memory): the stored-interior tiles stream from DRAM
// through shallow rings (1-2 stages), so they are warmed in L2 a few tiles ahead.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

namespace {

using namespace tc;

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int HD>
struct BwdCfg {
  static constexpr int ATOMS = (HD + 63) / 64;
  static constexpr int T128 = ATOMS * 128 * 128;  // 128-row tile bytes
  static constexpr int T64 = ATOMS * 64 * 128;    // 64-row tile bytes
  static constexpr int A128 = 128 * 128;          // atom stride, 128-row tile
  static constexpr int A64 = 64 * 128;            // atom stride, 64-row tile
  static constexpr int W_BYTES = 128 * 128;       // one [128 rows x 64] bf16 tile (1 atom)
};

// =====================================================================================
// dK, dV (+ keep bits)
// =====================================================================================
// STORED (no-recompute regime): Sᵀ is not recomputed; P = softmax_out and the dropout mask
// of each [64 queries x 128 keys] block come from the stored interior by TMA (2 stages), and
// P̃ = P·mask/(1-p) — the stored softmax_dropout_out by its definition (block.cpp:144-147) —
// is formed in registers, so the backward reads 3 of the 5 stored bytes per element.
template <int HD>
struct DkdvLayout {
  using C = BwdCfg<HD>;
  static constexpr int SMT = 64 * 128 * 2, MKT = 64 * 128;  // stored P / mask tiles
  template <bool STORED>
  struct L {
    // (Q, dO) ring depth: 3 stages keep the TMA of tile it+2 in flight while tile it's dV/dK
    // MMAs run (2 stages exposed the TMA latency between them); the stored variant needs its
    // smem for the P / mask tiles.
    // Recompute regimes keep P̃ᵀ and dSᵀ in TMEM (TS-form MMA), which frees the 64 KB of smem
    // the stored variant still uses for them; the (Q, dO) ring takes it.
    static constexpr int NS = HD > 128 ? (STORED ? 1 : 2) : (STORED ? 2 : 4);
    static constexpr int K_OFF = 0;
    static constexpr int V_OFF = STORED ? 0 : C::T128;
    static constexpr int QD_OFF = V_OFF + C::T128;
    static constexpr int W_OFF = QD_OFF + NS * 2 * C::T64;
    static constexpr int SMM_OFF = W_OFF + (STORED ? 4 * C::W_BYTES : 0);
    static constexpr int BAR_OFF = SMM_OFF + (STORED ? NS * (SMT + MKT) : 0);
    // [2 tiles][8 warps][32 queries] (log2 lse, rowdot) pairs, read as broadcasts
    static constexpr int STAT_OFF = BAR_OFF + 256;
    static constexpr int SMEM = STAT_OFF + 2 * 8 * 32 * 8 + 1024;
  };
};

// 32 x 32 bit transpose across a warp: lane r holds row r (bit c = column c) on entry and
// column r (bit c = row c) on exit; five butterfly rounds of one shuffle each.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  uint32_t m = 0x0000ffffu;
#pragma unroll
  for (int j = 16; j != 0; j >>= 1, m ^= m << j) {
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

template <int HD, bool CAUSAL, bool STORED>
// 320 threads = 3 warps on some SMSP (16 K registers each): 168 registers is the ceiling
// (__maxnreg__(200) compiles but fails to launch); the stored head_dim 160 variant spills.
__global__ void __launch_bounds__(320, 1)
    fa_bwd_dkdv_umma(const __grid_constant__ CUtensorMap map_kv,  // qkv, 128-row boxes
                     const __grid_constant__ CUtensorMap map_q,   // qkv, 64-row boxes
                     const __grid_constant__ CUtensorMap map_do,  // dO, 64-row boxes
                     const __grid_constant__ CUtensorMap map_sm,  // STORED: P, box {128 k, 64 q}
                     const __grid_constant__ CUtensorMap map_mk,  // STORED: mask, same box
                     AttnArgs a,
                     bf16* __restrict__ dqkv, const float* __restrict__ delta) {
  using C = BwdCfg<HD>;
  using Lay = typename DkdvLayout<HD>::template L<STORED>;
  constexpr int SMT = DkdvLayout<HD>::SMT, MKT = DkdvLayout<HD>::MKT;
  // smem: K, V (128 rows) | 2 x (Q, dO) (64 rows) | 2 x (P̃ᵀ, dSᵀ) (128 x 64) | [2 x (P, mask)]
  //       | lse/delta | bars        (STORED: no K)
  constexpr int K_OFF = Lay::K_OFF, V_OFF = Lay::V_OFF, QD_OFF = Lay::QD_OFF;
  constexpr int W_OFF = Lay::W_OFF, SMM_OFF = Lay::SMM_OFF;
  constexpr int BAR_OFF = Lay::BAR_OFF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  constexpr int NS = Lay::NS;
  uint64_t* kv_full = bar + 0;
  uint64_t* qd_full = bar + 1;          // [NS]
  uint64_t* qd_empty = bar + 1 + NS;    // [NS]
  uint64_t* sd_full = bar + 1 + 2 * NS; // [2] Sᵀ, dPᵀ ready in TMEM
  uint64_t* sd_free = sd_full + 2;      // [2] read by the warps
  uint64_t* w_full = sd_full + 4;       // [2] P̃ᵀ, dSᵀ written to smem
  uint64_t* w_free = sd_full + 6;       // [2] consumed by the dV/dK MMAs
  uint64_t* acc_full = sd_full + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sd_full + 9);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k0 = blockIdx.x * 128;
  const int hl = blockIdx.y / (int)a.b, bj = blockIdx.y % (int)a.b;
  const int S = (int)a.s;
  const int q_start = CAUSAL ? (k0 / 64) * 64 : 0;
  const int nq = (S - q_start + 63) / 64;
  const int kcol = (int)(a.koff + (int64_t)hl * HD), vcol = (int)(a.voff + (int64_t)hl * HD),
            qcol = (int)(a.qoff + (int64_t)hl * HD), dcol = hl * HD;
  const int64_t brow = ((int64_t)hl * a.b + bj) * a.s;
  // TMEM columns: Sᵀ [0,64) [64,128), dPᵀ [128,192) [192,256), dV [256,+HD), dK [384,+HD)
  // TMEM: Sᵀ and dPᵀ in SB buffers of 64 columns each, then dV and dK (HD columns each).
  // head_dim 160 single-buffers Sᵀ/dPᵀ to fit 64 + 64 + 160 + 160 <= 512 columns.
  constexpr int SB = HD > 128 ? 1 : 2;
  constexpr uint32_t S_COL = 0, DP_COL = SB * 64, DV_COL = 2 * SB * 64;
  constexpr uint32_t DK_COL = DV_COL + (HD > 128 ? HD : 128);

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&qd_full[i], 1);
      mbar_init(&qd_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sd_full[i], 1);
      mbar_init(&sd_free[i], 8);
      mbar_init(&w_full[i], 8);
      mbar_init(&w_free[i], 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc_warp(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(kv_full, (STORED ? 1 : 2) * C::T128);
#pragma unroll
      for (int at = 0; at < C::ATOMS; ++at) {
        if (!STORED) tma_load_3d(smem + K_OFF + at * C::A128, &map_kv, kv_full, kcol + 64 * at, bj, k0);
        tma_load_3d(smem + V_OFF + at * C::A128, &map_kv, kv_full, vcol + 64 * at, bj, k0);
      }
      for (int it = 0; it < nq; ++it) {
        const int st = it % NS;
        mbar_wait(&qd_empty[st], ((it / NS) & 1) ^ 1);
        uint8_t* Qt = smem + QD_OFF + st * 2 * C::T64;
        uint8_t* Dt = Qt + C::T64;
        const int qb = q_start + it * 64;
        mbar_expect_tx(&qd_full[st], 2 * C::T64 + (STORED ? SMT + MKT : 0));
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at) {
          tma_load_3d(Qt + at * C::A64, &map_q, &qd_full[st], qcol + 64 * at, bj, qb);
          tma_load_3d(Dt + at * C::A64, &map_do, &qd_full[st], dcol + 64 * at, bj, qb);
        }
        if (STORED) {
          uint8_t* St = smem + SMM_OFF + st * (SMT + MKT);
          tma_load_3d(St, &map_sm, &qd_full[st], k0, qb, (int)blockIdx.y);
          tma_load_3d(St + SMT, &map_mk, &qd_full[st], k0, qb, (int)blockIdx.y);
          for (int f = it == 0 ? 1 : 4; f <= 4 && it + f < nq; ++f) {  // warm L2 4 tiles ahead
            tma_prefetch_3d(&map_sm, k0, qb + 64 * f, (int)blockIdx.y);
            tma_prefetch_3d(&map_mk, k0, qb + 64 * f, (int)blockIdx.y);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_sd = make_idesc(128, 64, false, false);
      constexpr uint32_t idesc_acc = make_idesc(128, HD, false, true);
      const uint32_t ka = smem_u32(smem + K_OFF), va = smem_u32(smem + V_OFF);
      mbar_wait(kv_full, 0);
      auto issue_sd = [&](int it) {
        const int sb = it % SB, qs = it % NS;
        mbar_wait(&qd_full[qs], (it / NS) & 1);
        mbar_wait(&sd_free[sb], ((it / SB) & 1) ^ 1);
        tc_fence_after();
        const uint32_t qb = smem_u32(smem + QD_OFF + qs * 2 * C::T64), db = qb + C::T64;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t oa = (kk >> 2) * C::A128 + (kk & 3) * 32;
          const uint32_t ob = (kk >> 2) * C::A64 + (kk & 3) * 32;
          if (!STORED)
            umma_bf16(tmem + S_COL + sb * 64, desc_add(smem_desc(ka, 16, 1024), oa >> 4), desc_add(smem_desc(qb, 16, 1024), ob >> 4),
                      idesc_sd, kk > 0 ? 1u : 0u);
          umma_bf16(tmem + DP_COL + sb * 64, desc_add(smem_desc(va, 16, 1024), oa >> 4),
                    desc_add(smem_desc(db, 16, 1024), ob >> 4), idesc_sd, kk > 0 ? 1u : 0u);
        }
        umma_commit(&sd_full[sb]);
      };
      // look ahead one tile (Sᵀ/dPᵀ of it+1 before dV/dK of it) unless the (Q, dO) ring has a
      // single stage, where tile it+1 can only load after tile it's MMAs released it
      constexpr bool kAhead = NS > 1 && SB > 1;  // (single S/dP buffer: P̃ᵀ/dSᵀ live in it)
      if (nq > 0) issue_sd(0);
      for (int it = 0; it < nq; ++it) {
        if (kAhead && it + 1 < nq) issue_sd(it + 1);
        const int st = it & 1, qs = it % NS;
        mbar_wait(&w_full[st], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t pw = smem_u32(smem + W_OFF + st * 2 * C::W_BYTES), dw = pw + C::W_BYTES;
        const uint32_t qb = smem_u32(smem + QD_OFF + qs * 2 * C::T64), db = qb + C::T64;
        const int sb = it % SB;
#pragma unroll
        for (int kk = 0; kk < 64 / 16; ++kk) {
          // dV += P̃ᵀ·dO ; dK += dSᵀ·Q  (B = dO / Q tiles read MN-major)
          const uint64_t bdo = desc_add(smem_desc(db, C::A64, 1024), kk * (2048 >> 4));
          const uint64_t bq = desc_add(smem_desc(qb, C::A64, 1024), kk * (2048 >> 4));
          if constexpr (!STORED) {  // A from TMEM: queries 32h.. of half h at columns 32h..+16
            const uint32_t col = (uint32_t)(sb * 64 + (kk >> 1) * 32 + (kk & 1) * 8);
            umma_bf16_ts(tmem + DV_COL, tmem + S_COL + col, bdo, idesc_acc, (it | kk) != 0 ? 1u : 0u);
            umma_bf16_ts(tmem + DK_COL, tmem + DP_COL + col, bq, idesc_acc, (it | kk) != 0 ? 1u : 0u);
          } else {
            umma_bf16(tmem + DV_COL, desc_add(smem_desc(pw, 16, 1024), kk * 2), bdo, idesc_acc,
                      (it | kk) != 0 ? 1u : 0u);
            umma_bf16(tmem + DK_COL, desc_add(smem_desc(dw, 16, 1024), kk * 2), bq, idesc_acc,
                      (it | kk) != 0 ? 1u : 0u);
          }
        }
        umma_commit(&w_free[st]);
        umma_commit(&qd_empty[qs]);
        if (!kAhead && it + 1 < nq) issue_sd(it + 1);
      }
      umma_commit(acc_full);
    }
  } else {
    // ------------------------------------------------ softmax-backward warps
    const int qd = warp & 3;
    const int half = (warp - 2) >> 2;  // query columns 32*half .. +31 of each 64-query tile
    const int row = qd * 32 + lane;    // key row
    const int key = k0 + row;
    const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);
    const float sl2 = a.scale * kLog2e;
    const float inv_keep = a.drop.inv_keep;
    const bool drop_on = a.drop.thresh != 0;
    const int W = (S + 31) / 32;
    const uint32_t* kbits = a.keepbits;
    // lse (log2 domain), rowdot and the keep-bit word (q, this warp's 32 keys) of this half's
    // 32 queries of tile `it`: lane e holds query qb + 32*half + e. Loaded one tile ahead.
    auto row_stats = [&](int it, float& lse_o, float& dl_o, uint32_t& kw_o) {
      const int q = q_start + it * 64 + 32 * half + lane;
      lse_o = 0.f;
      kw_o = 0u;
      dl_o = (it < nq && q < S) ? delta[brow + q] : 0.f;
      if (!STORED && it < nq) {
        lse_o = q < S ? a.lse[brow + q] : INFINITY;  // scaled at use: keeps the load in flight
        kw_o = !drop_on ? 0xffffffffu
               : (q < S && (k0 >> 5) + qd < W) ? kbits[(brow + q) * W + (k0 >> 5) + qd] : 0u;
      }
    };
    float lse_n, dl_n;
    uint32_t kw_n;
    row_stats(0, lse_n, dl_n, kw_n);
    for (int it = 0; it < nq; ++it) {
      const int st = it & 1;
      const int qb = q_start + it * 64;
      const float lse_l = lse_n * kLog2e, dl_l = dl_n;
      const uint32_t kw_l = kw_n;
      row_stats(it + 1, lse_n, dl_n, kw_n);
      // this tile's row stats as smem broadcasts and the keep bits transposed to (this key,
      // the 32 queries): no per-element shuffles
      const bool shfl = a.stats_shfl != 0;
      // [-lse (log2) x 32 queries][-rowdot x 32 queries] of this warp, per tile parity
      float* stat = reinterpret_cast<float*>(smem + Lay::STAT_OFF) + ((it & 1) * 8 + (warp - 2)) * 64;
      uint32_t kt = 0u;
      if (!shfl) {
        stat[lane] = -lse_l;
        stat[32 + lane] = -dl_l;
        if constexpr (!STORED) kt = warp_transpose32(kw_l, lane);
        __syncwarp();
      }
      if (STORED) mbar_wait(&qd_full[it % NS], (it / NS) & 1);  // stored P / mask tiles landed
      const int sb = it % SB;
      mbar_wait(&sd_full[sb], (it / SB) & 1);
      tc_fence_after();
      uint32_t rs[32], rp[32];
      if (!STORED) tmem_ld32_nw(tl + S_COL + sb * 64 + half * 32, rs);
      tmem_ld32_nw(tl + DP_COL + sb * 64 + half * 32, rp);
      tmem_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sd_free[sb]);
      mbar_wait(&w_free[st], ((it >> 1) & 1) ^ 1);
      const int q0h = qb + 32 * half;
      uint32_t pw[16], dw[16];
      // interior tiles (every query and key in range, below the causal diagonal) skip the
      // per-element validity test
      const bool full = qb + 64 <= S && k0 + 128 <= S && !(CAUSAL && k0 + 127 > qb) &&
                        !a.masked_only;
      auto pd_loop = [&](auto masked) {
      constexpr bool kMasked = decltype(masked)::value;
      if constexpr (!STORED) {
        if (!shfl) {  // element pairs in packed fp32x2 arithmetic (same ops as the scalar form)
          const uint64_t sl2x2 = f32x2(sl2, sl2);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t nl2 = *reinterpret_cast<const uint64_t*>(stat + i);
            const uint64_t nd2 = *reinterpret_cast<const uint64_t*>(stat + 32 + i);
            float s0, s1;
            f32x2_split(ffma2(f32x2(__uint_as_float(rs[i]), __uint_as_float(rs[i + 1])), sl2x2, nl2),
                        s0, s1);
            float p0 = ex2(s0), p1 = ex2(s1);
            bool k0 = (kt >> i) & 1u, k1 = (kt >> (i + 1)) & 1u;
            if constexpr (kMasked) {
              const int qa = q0h + i, qb1 = q0h + i + 1;
              const bool v0 = qa < S && key < S && !(CAUSAL && key > qa);
              const bool v1 = qb1 < S && key < S && !(CAUSAL && key > qb1);
              p0 = v0 ? p0 : 0.f;
              p1 = v1 ? p1 : 0.f;
              k0 = k0 && v0;
              k1 = k1 && v1;
            }
            const uint64_t kf2 = f32x2(k0 ? inv_keep : 0.f, k1 ? inv_keep : 0.f);
            const uint64_t p2 = f32x2(p0, p1);
            float a0, a1, b0, b1;
            f32x2_split(fmul2(p2, kf2), a0, a1);
            f32x2_split(
                fmul2(p2, ffma2(f32x2(__uint_as_float(rp[i]), __uint_as_float(rp[i + 1])), kf2, nd2)),
                b0, b1);
            pw[i >> 1] = pack_bf16(a0, a1);
            dw[i >> 1] = pack_bf16(b0, b1);
          }
          return;
        }
      }
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float pv[2], dv[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int e = i + u;
          const int q = q0h + e;
          const bool valid = !kMasked || (q < S && key < S && !(CAUSAL && key > q));
          const float2 qs = shfl ? make_float2(0.f, 0.f) : make_float2(-stat[e], -stat[32 + e]);
          const float dqe = shfl ? __shfl_sync(0xffffffffu, dl_l, e) : qs.y;
          bool keep;
          float p;
          if constexpr (STORED) {
            // [64 q][128 k] tiles: this warp's 32 keys of query row 32*half + e
            const uint8_t* St = smem + SMM_OFF + (it % NS) * (SMT + MKT);
            const int qi = 32 * half + e;
            p = valid ? __bfloat162float(reinterpret_cast<const bf16*>(St)[qi * 128 + row]) : 0.f;
            keep = St[SMT + qi * 128 + row] != 0;
          } else {
            keep = shfl ? (__shfl_sync(0xffffffffu, kw_l, e) >> lane) & 1u : (kt >> e) & 1u;
            const float lqe = shfl ? __shfl_sync(0xffffffffu, lse_l, e) : qs.x;
            p = valid ? ex2(__uint_as_float(rs[e]) * sl2 - lqe) : 0.f;
          }
          keep = keep && valid;
          // P̃ = P·keep/(1-p); dS = P·(dP·keep/(1-p) - rowdot) with the keep factor selected
          // once and the dropout scale fused into the subtraction (4 instead of 6 FP ops)
          const float kf = keep ? inv_keep : 0.f;
          pv[u] = p * kf;
          dv[u] = p * fmaf(__uint_as_float(rp[e]), kf, -dqe);
        }
        pw[i >> 1] = pack_bf16(pv[0], pv[1]);
        dw[i >> 1] = pack_bf16(dv[0], dv[1]);
      }
      };
      if (full) pd_loop(std::false_type{});
      else pd_loop(std::true_type{});
      if constexpr (!STORED) {
        // P̃ᵀ / dSᵀ as bf16 pairs over the first 16 of this half's (consumed) 32 Sᵀ / dPᵀ columns
        tmem_st16u(tl + S_COL + sb * 64 + half * 32, pw);
        tmem_st16u(tl + DP_COL + sb * 64 + half * 32, dw);
        tmem_st_wait();
        tc_fence_before();
      } else {
        // [128 keys x 64 queries] K-major SW128 tiles: this half's queries = chunks 4h..4h+3
        uint8_t* prow = smem + W_OFF + st * 2 * C::W_BYTES + row * 128;
        uint8_t* drow = prow + C::W_BYTES;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int phys = (4 * half + u) ^ (row & 7);
          *reinterpret_cast<uint4*>(prow + phys * 16) =
              make_uint4(pw[4 * u], pw[4 * u + 1], pw[4 * u + 2], pw[4 * u + 3]);
          *reinterpret_cast<uint4*>(drow + phys * 16) =
              make_uint4(dw[4 * u], dw[4 * u + 1], dw[4 * u + 2], dw[4 * u + 3]);
        }
        fence_proxy_async();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&w_full[st]);
    }
    // epilogue: dK·scale, dV -> bf16 (halves take alternate 32-column chunks). Consecutive keys'
    // rows are b·ld elements apart: each warp stages its 32 rows of dK, then of dV, in the V
    // tile's shared memory (free: every MMA completed before acc_full; 16-byte chunks with the
    // low 3 chunk-index bits XOR-swizzled by row) and stores row-contiguous runs.
    mbar_wait(acc_full, 0);
    tc_fence_after();
    constexpr int CH = HD / 8;                       // 16-byte chunks per row
    constexpr int ORS = ((CH + 7) / 8) * 8 * 16;     // staging row stride (bytes)
    static_assert(C::T128 >= 128 * ORS, "epilogue staging");
    uint8_t* stg = smem + V_OFF + (row & ~31) * ORS;  // this warp's 32 rows
    const int nck = ((HD / 32 - half + 1) / 2) * 4;  // this half's chunks per row
    bf16* kbase = dqkv + ((int64_t)(k0 + (row & ~31)) * a.b + bj) * a.ld;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {  // dK, then dV
      const int col = pass == 0 ? DK_COL : DV_COL;
      const float sc = pass == 0 ? a.scale : 1.f;
#pragma unroll 1
      for (int c = half; c < HD / 32; c += 2) {
        float v[32];
        tmem_ld32(tl + col + c * 32, v);
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          const int ch = (c * 32 + i) / 8;
          *reinterpret_cast<uint4*>(stg + lane * ORS + (((ch & ~7) | ((ch & 7) ^ (lane & 7))) * 16)) =
              make_uint4(pack_bf16(v[i] * sc, v[i + 1] * sc), pack_bf16(v[i + 2] * sc, v[i + 3] * sc),
                         pack_bf16(v[i + 4] * sc, v[i + 5] * sc), pack_bf16(v[i + 6] * sc, v[i + 7] * sc));
        }
      }
      __syncwarp();
      const int dcol = pass == 0 ? kcol : vcol;
#pragma unroll 1
      for (int idx = lane; idx < 32 * nck; idx += 32) {
        const int r = idx / nck, k = idx % nck;
        const int ch = 4 * (half + 2 * (k >> 2)) + (k & 3);
        if (k0 + (row & ~31) + r < S)
          *reinterpret_cast<uint4*>(kbase + (int64_t)r * a.b * a.ld + dcol + ch * 8) =
              *reinterpret_cast<const uint4*>(stg + r * ORS + (((ch & ~7) | ((ch & 7) ^ (r & 7))) * 16));
      }
      __syncwarp();  // the staging rows are rewritten by the next pass
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, 512);
  }
}

// =====================================================================================
// dQ
// =====================================================================================
// STORED: S is not recomputed; P and the mask of each [128 queries x 64 keys] block come from
// the stored interior by TMA (P with the 128-byte swizzle, read conflict-free by row).
template <int HD>
struct DqLayout {
  using C = BwdCfg<HD>;
  static constexpr int SMT = 128 * 64 * 2, MKT = 128 * 64;
  template <bool STORED>
  struct L {
    // (K, V [, P, mask]) ring depth (head_dim 160: 48 KB K/V tiles leave room for fewer)
    // recompute regimes: dS in TMEM (TS-form MMA), its 32 KB of smem go to the ring
    static constexpr int NS = HD > 128 ? (STORED ? 1 : 2) : (STORED ? 2 : 5);
    static constexpr int Q_OFF = 0, D_OFF = C::T128, KV_OFF = 2 * C::T128;
    static constexpr int W_OFF = KV_OFF + NS * 2 * C::T64;
    static constexpr int SMM_OFF = W_OFF + (STORED ? 2 * C::W_BYTES : 0);
    static constexpr int BAR_OFF = SMM_OFF + (STORED ? NS * (SMT + MKT) : 0);
    static constexpr int SMEM = BAR_OFF + 256 + 1024;
  };
};

template <int HD, bool CAUSAL, bool STORED>
__global__ void __launch_bounds__(320, 1)
    fa_bwd_dq_umma(const __grid_constant__ CUtensorMap map_q,   // qkv, 128-row boxes
                   const __grid_constant__ CUtensorMap map_do,  // dO, 128-row boxes
                   const __grid_constant__ CUtensorMap map_kv,  // qkv, 64-row boxes
                   const __grid_constant__ CUtensorMap map_sm,  // STORED: P, box {64 k, 128 q}, SW128
                   const __grid_constant__ CUtensorMap map_mk,  // STORED: mask, same box
                   AttnArgs a,
                   bf16* __restrict__ dqkv, const float* __restrict__ delta) {
  using C = BwdCfg<HD>;
  using Lay = typename DqLayout<HD>::template L<STORED>;
  constexpr int SMT = DqLayout<HD>::SMT, MKT = DqLayout<HD>::MKT;
  // smem: Q, dO (128 rows) | 2 x (K, V) (64 rows) | 2 x dS (128 x 64) | [2 x (P, mask)] | bars
  constexpr int Q_OFF = Lay::Q_OFF, D_OFF = Lay::D_OFF, KV_OFF = Lay::KV_OFF;
  constexpr int W_OFF = Lay::W_OFF, SMM_OFF = Lay::SMM_OFF;
  constexpr int BAR_OFF = Lay::BAR_OFF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  constexpr int NS = Lay::NS;
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;          // [NS]
  uint64_t* kv_empty = bar + 1 + NS;    // [NS]
  uint64_t* sd_full = bar + 1 + 2 * NS; // [2]
  uint64_t* sd_free = sd_full + 2;      // [2]
  uint64_t* w_full = sd_full + 4;       // [2]
  uint64_t* w_free = sd_full + 6;       // [2]
  uint64_t* acc_full = sd_full + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sd_full + 9);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * 128;
  const int hl = blockIdx.y / (int)a.b, bj = blockIdx.y % (int)a.b;
  const int S = (int)a.s;
  const int kv_end = CAUSAL ? min(S, q0 + 128) : S;
  const int nkv = (kv_end + 63) / 64;
  const int kcol = (int)(a.koff + (int64_t)hl * HD), vcol = (int)(a.voff + (int64_t)hl * HD),
            qcol = (int)(a.qoff + (int64_t)hl * HD), dcol = hl * HD;
  const int64_t brow = ((int64_t)hl * a.b + bj) * a.s;
  constexpr uint32_t DQ_COL = 256;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sd_full[i], 1);
      mbar_init(&sd_free[i], 8);
      mbar_init(&w_full[i], 8);
      mbar_init(&w_free[i], 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc_warp(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, (STORED ? 1 : 2) * C::T128);
#pragma unroll
      for (int at = 0; at < C::ATOMS; ++at) {
        if (!STORED) tma_load_3d(smem + Q_OFF + at * C::A128, &map_q, q_full, qcol + 64 * at, bj, q0);
        tma_load_3d(smem + D_OFF + at * C::A128, &map_do, q_full, dcol + 64 * at, bj, q0);
      }
      for (int it = 0; it < nkv; ++it) {
        const int st = it % NS;
        mbar_wait(&kv_empty[st], ((it / NS) & 1) ^ 1);
        uint8_t* Kt = smem + KV_OFF + st * 2 * C::T64;
        uint8_t* Vt = Kt + C::T64;
        mbar_expect_tx(&kv_full[st], 2 * C::T64 + (STORED ? SMT + MKT : 0));
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at) {
          tma_load_3d(Kt + at * C::A64, &map_kv, &kv_full[st], kcol + 64 * at, bj, it * 64);
          tma_load_3d(Vt + at * C::A64, &map_kv, &kv_full[st], vcol + 64 * at, bj, it * 64);
        }
        if (STORED) {
          uint8_t* St = smem + SMM_OFF + st * (SMT + MKT);  // st = it % NS here
          tma_load_3d(St, &map_sm, &kv_full[st], it * 64, q0, (int)blockIdx.y);
          tma_load_3d(St + SMT, &map_mk, &kv_full[st], it * 64, q0, (int)blockIdx.y);
          for (int f = it == 0 ? 1 : 4; f <= 4 && it + f < nkv; ++f) {  // warm L2 4 tiles ahead
            tma_prefetch_3d(&map_sm, (it + f) * 64, q0, (int)blockIdx.y);
            tma_prefetch_3d(&map_mk, (it + f) * 64, q0, (int)blockIdx.y);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_sd = make_idesc(128, 64, false, false);
      constexpr uint32_t idesc_acc = make_idesc(128, HD, false, true);
      const uint32_t qa = smem_u32(smem + Q_OFF), da = smem_u32(smem + D_OFF);
      mbar_wait(q_full, 0);
      auto issue_sd = [&](int it) {
        const int st = it & 1, ks = it % NS;
        mbar_wait(&kv_full[ks], (it / NS) & 1);
        mbar_wait(&sd_free[st], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t kb = smem_u32(smem + KV_OFF + ks * 2 * C::T64), vb = kb + C::T64;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t oa = (kk >> 2) * C::A128 + (kk & 3) * 32;
          const uint32_t ob = (kk >> 2) * C::A64 + (kk & 3) * 32;
          if (!STORED)
            umma_bf16(tmem + st * 64, desc_add(smem_desc(qa, 16, 1024), oa >> 4), desc_add(smem_desc(kb, 16, 1024), ob >> 4),
                      idesc_sd, kk > 0 ? 1u : 0u);
          umma_bf16(tmem + 128 + st * 64, desc_add(smem_desc(da, 16, 1024), oa >> 4),
                    desc_add(smem_desc(vb, 16, 1024), ob >> 4), idesc_sd, kk > 0 ? 1u : 0u);
        }
        umma_commit(&sd_full[st]);
      };
      constexpr bool kAhead = NS > 1;  // see the dK/dV kernel
      if (nkv > 0) issue_sd(0);
      for (int it = 0; it < nkv; ++it) {
        if (kAhead && it + 1 < nkv) issue_sd(it + 1);
        const int st = it & 1, ks = it % NS;
        mbar_wait(&w_full[st], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t dsw = smem_u32(smem + W_OFF + st * C::W_BYTES);
        const uint32_t kb = smem_u32(smem + KV_OFF + ks * 2 * C::T64);
#pragma unroll
        for (int kk = 0; kk < 64 / 16; ++kk) {
          const uint64_t bk = desc_add(smem_desc(kb, C::A64, 1024), kk * (2048 >> 4));
          if constexpr (!STORED) {  // dS from TMEM: keys 32h.. of half h at columns 32h..+16
            const uint32_t col = (uint32_t)(st * 64 + (kk >> 1) * 32 + (kk & 1) * 8);
            umma_bf16_ts(tmem + DQ_COL, tmem + col, bk, idesc_acc, (it | kk) != 0 ? 1u : 0u);
          } else {
            umma_bf16(tmem + DQ_COL, desc_add(smem_desc(dsw, 16, 1024), kk * 2), bk, idesc_acc,
                      (it | kk) != 0 ? 1u : 0u);
          }
        }
        umma_commit(&w_free[st]);
        umma_commit(&kv_empty[ks]);
        if (!kAhead && it + 1 < nkv) issue_sd(it + 1);
      }
      umma_commit(acc_full);
    }
  } else {
    const int qd = warp & 3;
    const int half = (warp - 2) >> 2;  // key columns 32*half .. +31 of each 64-key tile
    const int row = qd * 32 + lane;    // query row
    const int qr = q0 + row;
    const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);
    const float sl2 = a.scale * kLog2e;
    const float inv_keep = a.drop.inv_keep;
    const bool drop_on = a.drop.thresh != 0;
    const int W = (S + 31) / 32;
    const float lse2 = (!STORED && qr < S) ? a.lse[brow + qr] * kLog2e : INFINITY;
    const float dl = qr < S ? delta[brow + qr] : 0.f;
    const uint32_t* kb = STORED ? nullptr : a.keepbits + (brow + (qr < S ? qr : 0)) * W;
    auto key_word = [&](int it) {  // keep bits of (this row, keys it*64 + 32*half ..)
      const int kc = it * 64 + 32 * half;
      return (STORED || !drop_on) ? 0xffffffffu : (it < nkv && qr < S && kc < S) ? kb[kc >> 5] : 0u;
    };
    uint32_t word_n = key_word(0);
    for (int it = 0; it < nkv; ++it) {
      const int st = it & 1;
      const int kc0 = it * 64 + 32 * half;
      uint32_t word = word_n;
      word_n = key_word(it + 1);
      uint32_t pst[16];  // STORED: this half's 32 stored probabilities (bf16 pairs)
      if constexpr (STORED) {
        mbar_wait(&kv_full[it % NS], (it / NS) & 1);  // stored P / mask tiles landed
        const uint8_t* St = smem + SMM_OFF + (it % NS) * (SMT + MKT);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint4 v = *reinterpret_cast<const uint4*>(St + row * 128 + (((4 * half + u) ^ (row & 7)) * 16));
          pst[4 * u] = v.x; pst[4 * u + 1] = v.y; pst[4 * u + 2] = v.z; pst[4 * u + 3] = v.w;
        }
        const uint4 m0 = *reinterpret_cast<const uint4*>(St + SMT + row * 64 + 32 * half);
        const uint4 m1 = *reinterpret_cast<const uint4*>(St + SMT + row * 64 + 32 * half + 16);
        const uint32_t mw[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
        word = 0u;
#pragma unroll
        for (int e = 0; e < 32; ++e) word |= ((mw[e >> 2] >> (8 * (e & 3))) & 1u) << e;
      }
      mbar_wait(&sd_full[st], (it >> 1) & 1);
      tc_fence_after();
      uint32_t rs[32], rp[32];
      if (!STORED) tmem_ld32_nw(tl + st * 64 + half * 32, rs);
      tmem_ld32_nw(tl + 128 + st * 64 + half * 32, rp);
      tmem_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sd_free[st]);
      mbar_wait(&w_free[st], ((it >> 1) & 1) ^ 1);
      const bool full = kc0 + 32 <= S && !(CAUSAL && kc0 + 31 > q0) && q0 + 128 <= S &&
                        !a.masked_only;
      uint32_t dw[16];
      // two copies of the element loop: interior tiles skip the per-element bounds / causal test
      auto ds_loop = [&](auto masked) {
        constexpr bool kMasked = decltype(masked)::value;
        if constexpr (!STORED) {  // element pairs in packed fp32x2 arithmetic (bit-identical)
          const uint64_t sl2x2 = f32x2(sl2, sl2), nl2 = f32x2(-lse2, -lse2),
                         nd2 = f32x2(-dl, -dl);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float s0, s1;
            f32x2_split(ffma2(f32x2(__uint_as_float(rs[i]), __uint_as_float(rs[i + 1])), sl2x2, nl2),
                        s0, s1);
            float p0 = ex2(s0), p1 = ex2(s1);
            if (kMasked && (kc0 + i >= S || qr >= S || (CAUSAL && kc0 + i > qr))) p0 = 0.f;
            if (kMasked && (kc0 + i + 1 >= S || qr >= S || (CAUSAL && kc0 + i + 1 > qr))) p1 = 0.f;
            const uint64_t kf2 = f32x2((word >> i) & 1u ? inv_keep : 0.f,
                                       (word >> (i + 1)) & 1u ? inv_keep : 0.f);
            float d0, d1;
            f32x2_split(fmul2(f32x2(p0, p1), ffma2(f32x2(__uint_as_float(rp[i]),
                                                         __uint_as_float(rp[i + 1])), kf2, nd2)),
                        d0, d1);
            dw[i >> 1] = pack_bf16(d0, d1);
          }
        } else {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float dv[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int e = i + u;
            const bool keep = (word >> e) & 1u;
            float p;
            if constexpr (STORED)
              p = __uint_as_float((e & 1) ? (pst[e >> 1] & 0xffff0000u) : (pst[e >> 1] << 16));
            else
              p = ex2(__uint_as_float(rs[e]) * sl2 - lse2);
            if (kMasked && (kc0 + e >= S || qr >= S || (CAUSAL && kc0 + e > qr))) p = 0.f;
            const float kf = keep ? inv_keep : 0.f;  // see the dK/dV kernel
            dv[u] = p * fmaf(__uint_as_float(rp[e]), kf, -dl);
          }
          dw[i >> 1] = pack_bf16(dv[0], dv[1]);
        }
        }
      };
      if (full) ds_loop(std::false_type{});
      else ds_loop(std::true_type{});
      if constexpr (!STORED) {
        tmem_st16u(tl + st * 64 + half * 32, dw);  // over this half's consumed S columns
        tmem_st_wait();
        tc_fence_before();
      } else {
        uint8_t* drow = smem + W_OFF + st * C::W_BYTES + row * 128;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int phys = (4 * half + u) ^ (row & 7);
          *reinterpret_cast<uint4*>(drow + phys * 16) =
              make_uint4(dw[4 * u], dw[4 * u + 1], dw[4 * u + 2], dw[4 * u + 3]);
        }
        fence_proxy_async();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&w_full[st]);
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    bf16* out = dqkv + ((int64_t)(qr < S ? qr : 0) * a.b + bj) * a.ld + qcol;
#pragma unroll 1
    for (int c = half; c < HD / 32; c += 2) {
      float v[32];
      tmem_ld32(tl + DQ_COL + c * 32, v);
      if (qr < S) {
        const float sc = a.scale;
        if ((((uintptr_t)(out + c * 32)) & 31) == 0) {  // full 32-byte sectors per lane
#pragma unroll
          for (int i = 0; i < 32; i += 16)
            st_v8(out + c * 32 + i, pack_bf16(v[i] * sc, v[i + 1] * sc), pack_bf16(v[i + 2] * sc, v[i + 3] * sc),
                  pack_bf16(v[i + 4] * sc, v[i + 5] * sc), pack_bf16(v[i + 6] * sc, v[i + 7] * sc),
                  pack_bf16(v[i + 8] * sc, v[i + 9] * sc), pack_bf16(v[i + 10] * sc, v[i + 11] * sc),
                  pack_bf16(v[i + 12] * sc, v[i + 13] * sc), pack_bf16(v[i + 14] * sc, v[i + 15] * sc));
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 8)
            *reinterpret_cast<uint4*>(out + c * 32 + i) = make_uint4(
                pack_bf16(v[i] * sc, v[i + 1] * sc), pack_bf16(v[i + 2] * sc, v[i + 3] * sc),
                pack_bf16(v[i + 4] * sc, v[i + 5] * sc), pack_bf16(v[i + 6] * sc, v[i + 7] * sc));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, 512);
  }
}

}  // namespace

// 3-D map over a stored interior {nblk = lh*b, s, s} (row = query, contiguous keys):
// dims {s (key), s (query), nblk}; box {box_k, box_q, 1}. Also used by the fused backward.
CUtensorMap interior_map(const void* ptr, bool u8, int64_t s, int64_t nblk, int box_k, int box_q,
                         bool sw128) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  const int64_t es = u8 ? 1 : 2;
  const cuuint64_t dims[3] = {(cuuint64_t)s, (cuuint64_t)s, (cuuint64_t)nblk};
  const cuuint64_t strides[2] = {(cuuint64_t)(s * es), (cuuint64_t)(s * s * es)};
  const cuuint32_t box[3] = {(cuuint32_t)box_k, (cuuint32_t)box_q, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn_bwd()(&m, u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                               3, const_cast<void*>(ptr), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE,
                               sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(3, "cuTensorMapEncodeTiled (interior) failed: " + std::to_string((int)r));
  return m;
}

namespace {

template <int HD, bool CAUSAL, bool STORED>
void launch_bwd_umma(const AttnArgs& a, const bf16* dout, bf16* dqkv, const float* delta,
                     cudaStream_t st) {
  constexpr int smem_kv = DkdvLayout<HD>::template L<STORED>::SMEM;
  constexpr int smem_q = DqLayout<HD>::template L<STORED>::SMEM;
  static_assert(smem_kv <= 232448 && smem_q <= 232448, "attention backward: smem over the limit");
  static bool once = [] {
    SPL_CUDA(cudaFuncSetAttribute(fa_bwd_dkdv_umma<HD, CAUSAL, STORED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv));
    SPL_CUDA(cudaFuncSetAttribute(fa_bwd_dq_umma<HD, CAUSAL, STORED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q));
    return true;
  }();
  (void)once;
  const CUtensorMap m128 = attn_seq_map(a.qkv, a.ld, a.b, a.s, a.ld, 128);
  const CUtensorMap m64 = attn_seq_map(a.qkv, a.ld, a.b, a.s, a.ld, 64);
  const CUtensorMap d64 = attn_seq_map(dout, a.ldo, a.b, a.s, a.ldo, 64);
  const CUtensorMap d128 = attn_seq_map(dout, a.ldo, a.b, a.s, a.ldo, 128);
  CUtensorMap skv = m128, mkv = m128, sq = m128, mq = m128;  // unused unless STORED
  if (STORED) {
    const int64_t nblk = a.lh * a.b;
    skv = interior_map(a.sm, false, a.s, nblk, 128, 64, false);
    mkv = interior_map(a.mask, true, a.s, nblk, 128, 64, false);
    sq = interior_map(a.sm, false, a.s, nblk, 64, 128, true);
    mq = interior_map(a.mask, true, a.s, nblk, 64, 128, false);
  }
  dim3 grid((unsigned)((a.s + 127) / 128), (unsigned)(a.lh * a.b));
  // dK/dV: K,V 128-row boxes + Q 64-row boxes from the same map family
  fa_bwd_dkdv_umma<HD, CAUSAL, STORED><<<grid, 320, smem_kv, st>>>(m128, m64, d64, skv, mkv, a, dqkv, delta);
  SPL_CHECK_LAUNCH();
  fa_bwd_dq_umma<HD, CAUSAL, STORED><<<grid, 320, smem_q, st>>>(m128, d128, m64, sq, mq, a, dqkv, delta);
  SPL_CHECK_LAUNCH();
}

}  // namespace

bool attn_bwd_umma_supported(const AttnArgs& a) {
  const bool hd_ok = a.hd == 64 || a.hd == 96 || a.hd == 128 || a.hd == 160;
  const bool regime_ok =
      a.sm == nullptr ? (a.lse != nullptr && (a.keepbits != nullptr || a.drop.thresh == 0))
                      : (a.mask != nullptr && a.s % 64 == 0 && ((uintptr_t)a.sm & 15) == 0 &&
                         ((uintptr_t)a.mask & 15) == 0);
  return hd_ok && regime_ok && a.ld % 8 == 0 && a.ldo % 8 == 0 && ((uintptr_t)a.qkv & 15) == 0 &&
         ((uintptr_t)a.o & 15) == 0 && a.s < (1 << 30);
}

void attn_bwd_umma(const AttnArgs& a_in, const void* dout, void* dqkv, const float* delta,
                   cudaStream_t st) {
  static const int masked_only = [] {
    const char* e = std::getenv("SPL_ATTN_MASKED_ONLY");
    return (e != nullptr && e[0] == '1') ? 1 : 0;
  }();
  static const int stats_shfl = [] {
    const char* e = std::getenv("SPL_ATTN_SHFL");
    return (e != nullptr && e[0] == '1') ? 1 : 0;
  }();
  AttnArgs a = a_in;
  a.masked_only = masked_only;
  a.stats_shfl = stats_shfl;
  const bf16* d = static_cast<const bf16*>(dout);
  bf16* g = static_cast<bf16*>(dqkv);
#define SPL_BWD_CASE(HDX)                                                                        \
  case HDX:                                                                                      \
    if (a.sm != nullptr)                                                                         \
      return a.causal ? launch_bwd_umma<HDX, true, true>(a, d, g, delta, st)                     \
                      : launch_bwd_umma<HDX, false, true>(a, d, g, delta, st);                   \
    return a.causal ? launch_bwd_umma<HDX, true, false>(a, d, g, delta, st)                      \
                    : launch_bwd_umma<HDX, false, false>(a, d, g, delta, st);
  switch (a.hd) {
    SPL_BWD_CASE(64)
    SPL_BWD_CASE(96)
    SPL_BWD_CASE(128)
    SPL_BWD_CASE(160)
    default: raise(3, "attn_bwd_umma: unsupported head_dim");
  }
#undef SPL_BWD_CASE
}

}  // namespace spl::k
