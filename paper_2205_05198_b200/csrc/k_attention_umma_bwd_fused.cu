// Attention backward in ONE kernel per (key block, head, batch) for the recompute regimes
// (selective / full), tcgen05 + TMEM + TMA, bf16, head_dim 64 / 96: dK, dV and dQ from a single
// recomputation of Sᵀ, dPᵀ and the softmax-backward elements (block.cpp:159-193), where the
// split kernels (k_attention_umma_bwd.cu) recompute them twice (7 GEMM-equivalents and two
// exponentials per element instead of 5 and one).
//
// CTA = 128 keys of one (head, batch), loops over 64-query tiles (the dK/dV kernel's loop):
//   MMA   Sᵀ = K·Qᵀ, dPᵀ = V·dOᵀ (M=128 keys, N=64 queries, SS)          -> TMEM (2 buffers)
//   warps Pᵀ = exp2(Sᵀc - lse), keep from the keep bits (transposed per warp),
//         P̃ᵀ = Pᵀ·keep/(1-p) -> TMEM over the consumed Sᵀ columns (A of a TS-form MMA),
//         dSᵀ = Pᵀ∘(dPᵀ·keep/(1-p) - rowdot) -> smem, bf16 [128 keys][64 queries] SW128
//   MMA   dV += P̃ᵀ·dO, dK += dSᵀ·Q (TS: dSᵀ also written to TMEM over the consumed dPᵀ),
//         dQᵀ = Kᵀ·dSᵀ (SS: M = head_dim rows padded to 128 read MN-major from the K tile,
//         B = the same dSᵀ tile read MN-major) -> TMEM (its own 64 columns)
//   warps dQ readers (one per 32 head_dim rows) add the dQᵀ tile into an fp32 accumulator
//         dq_acc[(head, batch)][query][head_dim] with red.global.add.f32 (coalesced: lanes =
//         consecutive head_dim), so the dQ sum over key blocks happens in L2 (order between
//         key blocks is not fixed: dQ is reproducible to fp32 rounding, dK / dV bit-exactly;
//         SPL_ATTN_DETERMINISTIC=1 selects the split kernels).
// fa_bwd_prep (before): rowdot -> -rowdot, -lse·log2(e) per query row (loaded per tile by
// the producer with bulk copies) and zeroes dq_acc; fa_bwd_dq_store (after): dq_acc·scale ->
// bf16 into the Q columns of dqkv.
//
// Warp roles (512 threads, 128 registers each):
//   warps 0-7   softmax-backward elements (TMEM lane quadrant = warp & 3; warps 0-3 the even,
//               4-7 the odd query tiles, in ping-pong)
//   warps 8-11  dQ readers (TMEM lane quadrant = warp & 3; idle when 32·quadrant >= head_dim)
//   warp 12     TMA producer; warp 13 TMEM allocator + MMA issuer; warps 14-15 idle
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace spl::k {

CUtensorMap attn_seq_map(const void* ptr, int64_t width, int64_t b, int64_t s, int64_t ld, int rows);
CUtensorMap interior_map(const void* ptr, bool u8, int64_t s, int64_t nblk, int box_k, int box_q,
                         bool sw128);

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
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a TMA box (no shared memory, no barrier): the stored-interior tiles come from
// DRAM, and the 2-stage ring alone leaves their latency exposed.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  uint32_t m = 0x0000ffffu;
#pragma unroll
  for (int j = 16; j != 0; j >>= 1, m ^= m << j) {
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

// SPL_ATTN_TRACE=1 (dev A/B): clock64() stamps of one CTA's pipeline events, printed after
// the first launch — [event][tile]
__device__ unsigned long long* g_trace = nullptr;
constexpr int kTraceX = 3, kTraceY = 100;
#define TRACE(e, it)                                                                         \
  do {                                                                                       \
    if (tr != nullptr && (it) < 64) tr[(e) * 64 + (it)] = (unsigned long long)clock64();     \
  } while (0)

// STORED (no-recompute regime): Sᵀ is not recomputed — P = softmax_out and the dropout mask
// of each [64 queries x 128 keys] block are loaded by TMA from the stored interior into the
// Q / dO ring stage (3 of the 5 stored bytes per element read once), P̃ = P·keep/(1-p).
template <int HD, bool STORED = false>
struct FusedCfg {
  static_assert(HD == 64 || HD == 96, "fused attention backward: head_dim 64 or 96");
  static constexpr int ATOMS = (HD + 63) / 64;
  static constexpr int A128 = 128 * 128;        // atom stride of a 128-row tile
  static constexpr int A64 = 64 * 128;          // atom stride of a 64-row tile
  static constexpr int T128 = ATOMS * A128;
  static constexpr int T64 = ATOMS * A64;
  // (Q, dO, stats) ring depth (a stage is released when the dV/dK MMAs of its tile complete)
  static constexpr int NS = STORED ? 2 : (HD > 64 ? 3 : 5);
  static constexpr int K_OFF = 0, V_OFF = T128, QD_OFF = 2 * T128;
  static constexpr int ST_OFF = QD_OFF + NS * 2 * T64;          // [NS][-lse·log2e x64][-rowdot x64]
  // dSᵀ [2 tile parities][128 x 64 bf16]
  static constexpr int DS_OFF = (ST_OFF + NS * 512 + 1023) / 1024 * 1024;
  static constexpr int DS_BYTES = 128 * 128;
  static constexpr int PM_OFF = DS_OFF + 2 * DS_BYTES;            // STORED: [NS][P | mask]
  static constexpr int P_TILE = 64 * 128 * 2, M_TILE = 64 * 128, PM_STAGE = P_TILE + M_TILE;
  static constexpr int BAR_OFF = PM_OFF + (STORED ? NS * PM_STAGE : 0);
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  // TMEM: Sᵀ [0,128) (2 x 64), dPᵀ [128,256), dV, dK (HD each), dQᵀ (64)
  static constexpr uint32_t S_COL = 0, DP_COL = 128, DV_COL = 256, DK_COL = 256 + HD;
  static constexpr uint32_t DQ_COL = 256 + 2 * HD;
  static_assert(DQ_COL + 64 <= 512, "TMEM budget");
  static constexpr int NQW = (HD + 31) / 32;  // dQ reader warps
};

template <int HD, bool CAUSAL, bool KT, bool STORED>
__global__ void __launch_bounds__(512, 1)
    fa_bwd_fused_umma(const __grid_constant__ CUtensorMap map_kv,  // qkv, 128-row boxes
                      const __grid_constant__ CUtensorMap map_q,   // qkv, 64-row boxes
                      const __grid_constant__ CUtensorMap map_do,  // dO, 64-row boxes
                      const __grid_constant__ CUtensorMap map_sm,  // STORED: P, box {128 k, 64 q}
                      const __grid_constant__ CUtensorMap map_mk,  // STORED: mask, same box
                      AttnArgs a, bf16* __restrict__ dqkv) {
  using C = FusedCfg<HD, STORED>;
  constexpr int NS = C::NS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* kv_full = bar + 0;
  uint64_t* qd_full = bar + 1;           // [NS]
  uint64_t* qd_empty = bar + 1 + NS;     // [NS]
  uint64_t* sd_full = bar + 1 + 2 * NS;  // [2] Sᵀ, dPᵀ in TMEM
  uint64_t* sd_free = sd_full + 2;       // [2] read by the softmax warps
  uint64_t* w_full = sd_full + 4;        // [2] P̃ᵀ (TMEM) + dSᵀ (smem) written
  uint64_t* w_free = sd_full + 6;        // [2] consumed by the dV / dK / dQᵀ MMAs
  uint64_t* dq_full = sd_full + 8;       // dQᵀ of the current tile in TMEM
  uint64_t* dq_free = sd_full + 9;       // read out by the dQ readers
  uint64_t* acc_full = sd_full + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sd_full + 11);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k0 = blockIdx.x * 128;
  const int hb = blockIdx.y;
  const int hl = hb / (int)a.b, bj = hb % (int)a.b;
  const int S = (int)a.s;
  const int q_start = CAUSAL ? (k0 / 64) * 64 : 0;
  const int nq = (S - q_start) / 64;
  const int kcol = (int)(a.koff + (int64_t)hl * HD), vcol = (int)(a.voff + (int64_t)hl * HD),
            qcol = (int)(a.qoff + (int64_t)hl * HD), dcol = hl * HD;
  const int64_t brow = (int64_t)hb * a.s;
  const float* nlse = a.bstat;                  // -lse·log2(e)  [lh*b*s]
  const float* ndel = a.bstat + a.lh * a.b * a.s;  // -rowdot

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&qd_full[i], 1);
      mbar_init(&qd_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sd_full[i], 1);
      mbar_init(&sd_free[i], 4);
      mbar_init(&w_full[i], 4);
      mbar_init(&w_free[i], 1);
    }
    mbar_init(dq_full, 1);
    mbar_init(dq_free, C::NQW);
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 13) tmem_alloc_warp(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  unsigned long long* tr =
      (g_trace != nullptr && blockIdx.x == kTraceX && blockIdx.y == kTraceY) ? g_trace : nullptr;
  if (threadIdx.x == 0) TRACE(15, 0);

  if (warp >= 12) {
    if (warp == 12 && lane == 0) {
      // ------------------------------------------------ TMA producer
      mbar_expect_tx(kv_full, 2 * C::T128);
#pragma unroll
      for (int at = 0; at < C::ATOMS; ++at) {
        tma_load_3d(smem + C::K_OFF + at * C::A128, &map_kv, kv_full, kcol + 64 * at, bj, k0);
        tma_load_3d(smem + C::V_OFF + at * C::A128, &map_kv, kv_full, vcol + 64 * at, bj, k0);
      }
      for (int it = 0; it < nq; ++it) {
        const int st = it % NS;
        mbar_wait(&qd_empty[st], ((it / NS) & 1) ^ 1);
        TRACE(13, it);
        uint8_t* Qt = smem + C::QD_OFF + st * 2 * C::T64;
        uint8_t* Dt = Qt + C::T64;
        float* stt = reinterpret_cast<float*>(smem + C::ST_OFF + st * 512);
        const int qb = q_start + it * 64;
        mbar_expect_tx(&qd_full[st], 2 * C::T64 + 512 + (STORED ? C::PM_STAGE : 0));
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at) {
          tma_load_3d(Qt + at * C::A64, &map_q, &qd_full[st], qcol + 64 * at, bj, qb);
          tma_load_3d(Dt + at * C::A64, &map_do, &qd_full[st], dcol + 64 * at, bj, qb);
        }
        if constexpr (STORED) {  // P and mask of (these 64 queries, the CTA's 128 keys)
          uint8_t* pm = smem + C::PM_OFF + st * C::PM_STAGE;
          tma_load_3d(pm, &map_sm, &qd_full[st], k0, qb, hb);
          tma_load_3d(pm + C::P_TILE, &map_mk, &qd_full[st], k0, qb, hb);
          if (it == 0)  // warm L2 with the tiles the ring reaches next
            for (int f = 1; f < 4 && f < nq; ++f) {
              tma_prefetch_3d(&map_sm, k0, qb + 64 * f, hb);
              tma_prefetch_3d(&map_mk, k0, qb + 64 * f, hb);
            }
          if (it + 4 < nq) {
            tma_prefetch_3d(&map_sm, k0, qb + 256, hb);
            tma_prefetch_3d(&map_mk, k0, qb + 256, hb);
          }
        }
        bulk_load(stt, nlse + brow + qb, 256, &qd_full[st]);
        bulk_load(stt + 64, ndel + brow + qb, 256, &qd_full[st]);
      }
    } else if (warp == 13) {
      // ------------------------------------------------ MMA issuer (whole warp, elected lane)
      constexpr uint32_t idesc_sd = make_idesc(128, 64, false, false);
      constexpr uint32_t idesc_acc = make_idesc(128, HD, false, true);
      constexpr uint32_t idesc_dq = make_idesc(128, 64, true, true);
      const uint32_t ka = smem_u32(smem + C::K_OFF), va = smem_u32(smem + C::V_OFF);
      const uint64_t kd0 = smem_desc(ka, 16, 1024), vd0 = smem_desc(va, 16, 1024);
      const uint64_t kdq = smem_desc(ka, C::A128, 1024);
      mbar_wait(kv_full, 0);
      auto issue_sd = [&](int it) {
        const int sb = it & 1, qs = it % NS;
        if (lane == 0) TRACE(0, it);
        mbar_wait(&qd_full[qs], (it / NS) & 1);
        mbar_wait(&sd_free[sb], ((it >> 1) & 1) ^ 1);
        if (lane == 0) TRACE(1, it);
        tc_fence_after();
        const uint32_t qb = smem_u32(smem + C::QD_OFF + qs * 2 * C::T64), db = qb + C::T64;
        // descriptors built once; each K step advances the start-address field (desc_add)
        const uint64_t qd = smem_desc(qb, 16, 1024), dd = smem_desc(db, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t oa = ((kk >> 2) * C::A128 + (kk & 3) * 32) >> 4;
          const uint32_t ob = ((kk >> 2) * C::A64 + (kk & 3) * 32) >> 4;
          if constexpr (!STORED)
            umma_bf16_w(tmem + C::S_COL + sb * 64, desc_add(kd0, oa), desc_add(qd, ob), idesc_sd,
                        kk > 0 ? 1u : 0u);
          umma_bf16_w(tmem + C::DP_COL + sb * 64, desc_add(vd0, oa), desc_add(dd, ob), idesc_sd,
                      kk > 0 ? 1u : 0u);
        }
        umma_commit_w(&sd_full[sb]);
      };
      if (nq > 0) issue_sd(0);
      for (int it = 0; it < nq; ++it) {
        if (it + 1 < nq) issue_sd(it + 1);
        const int st = it & 1, qs = it % NS;
        mbar_wait(&w_full[st], (it >> 1) & 1);
        if (lane == 0) TRACE(2, it);
        tc_fence_after();
        const uint32_t dsw = smem_u32(smem + C::DS_OFF + st * C::DS_BYTES);
        const uint64_t dsd = smem_desc(dsw, 8192, 1024);
        const uint32_t qb = smem_u32(smem + C::QD_OFF + qs * 2 * C::T64), db = qb + C::T64;
        const uint64_t dd = smem_desc(db, C::A64, 1024), qd = smem_desc(qb, C::A64, 1024);
#pragma unroll
        for (int kk = 0; kk < 64 / 16; ++kk) {
          // dV += P̃ᵀ·dO, dK += dSᵀ·Q (A: P̃ᵀ / dSᵀ in TMEM, queries 32h.. of half h at
          // columns 32h..+16)
          const uint64_t bdo = desc_add(dd, kk * (2048 >> 4));
          const uint64_t bq = desc_add(qd, kk * (2048 >> 4));
          const uint32_t col = (uint32_t)(st * 64 + (kk >> 1) * 32 + (kk & 1) * 8);
          umma_bf16_ts_w(tmem + C::DV_COL, tmem + C::S_COL + col, bdo, idesc_acc, (it | kk) != 0 ? 1u : 0u);
          umma_bf16_ts_w(tmem + C::DK_COL, tmem + C::DP_COL + col, bq, idesc_acc, (it | kk) != 0 ? 1u : 0u);
        }
        umma_commit_w(&qd_empty[qs]);  // the stage's Q / dO are read by now
        // dQᵀ = Kᵀ·dSᵀ: K = the CTA's 128 keys in 8 steps of 16 rows; A = K tile MN-major
        // (head_dim rows, padded to M = 128), B = dSᵀ MN-major (queries contiguous)
        mbar_wait(dq_free, ((it & 1) ^ 1));
        if (lane == 0) TRACE(3, it);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          umma_bf16_w(tmem + C::DQ_COL, desc_add(kdq, kk * (2048 >> 4)),
                      desc_add(dsd, kk * (2048 >> 4)), idesc_dq, kk > 0 ? 1u : 0u);
        umma_commit_w(&w_free[st]);
        umma_commit_w(dq_full);
        if (lane == 0) TRACE(4, it);
      }
      umma_commit_w(acc_full);
    }
  } else if (warp >= 8) {
    // ------------------------------------------------ dQ readers
    const int qd = warp & 3;
    if (qd < C::NQW) {
      const int row = qd * 32 + lane;  // head_dim index
      const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16) + C::DQ_COL;
      float* accp = a.dq_acc + (brow + q_start) * HD + row;
      for (int it = 0; it < nq; ++it) {
        mbar_wait(dq_full, it & 1);
        if (lane == 0 && qd == 0) TRACE(10, it);
        tc_fence_after();
        uint32_t v0[32], v1[32];
        tmem_ld32_nw(tl, v0);
        tmem_ld32_nw(tl + 32, v1);
        tmem_wait();
        if (lane == 0 && qd == 0) TRACE(11, it);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dq_free);
        if (row < HD) {
          float* p = accp + (int64_t)it * 64 * HD;
#pragma unroll
          for (int c = 0; c < 32; ++c)
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p + c * HD), "f"(__uint_as_float(v0[c])) : "memory");
#pragma unroll
          for (int c = 0; c < 32; ++c)
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p + (32 + c) * HD), "f"(__uint_as_float(v1[c])) : "memory");
        }
        if (lane == 0 && qd == 0) TRACE(12, it);
      }
    }
  } else {
    // ------------------------------------------------ softmax-backward warps
    // Two warpgroups in ping-pong: warps 0-3 take the even query tiles (Sᵀ/dPᵀ buffer 0),
    // warps 4-7 the odd ones (buffer 1), each warp all 64 queries of its key row in two
    // 32-query halves — so one group's TMEM loads (64 KB of fp32 Sᵀ/dPᵀ per tile, the TMEM
    // read port is the narrowest resource) overlap the other group's element work.
    const int qd = warp & 3;
    const int wg = warp >> 2;         // tile parity
    const int row = qd * 32 + lane;   // key row
    const int key = k0 + row;
    const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);
    const float sl2 = a.scale * kLog2e;
    const float inv_keep = a.drop.inv_keep;
    const bool drop_on = a.drop.thresh != 0;
    const int W = S / 32;
    const uint32_t* kbits = a.keepbits;
    // keep bits of (this key, the 32 queries of half h of tile it): KT reads the transposed
    // layout directly; otherwise each lane loads (its query, the warp's 32 keys) and the warp
    // transposes the 32 x 32 block. Loaded one own tile ahead.
    auto kword = [&](int it, int h) -> uint32_t {
      if (STORED || !drop_on) return 0xffffffffu;
      if (it >= nq) return 0u;
      const int qw = (q_start + it * 64 + 32 * h) >> 5;
      if constexpr (KT) return kbits[((int64_t)hb * (S >> 5) + qw) * S + key];
      return kbits[(brow + 32 * qw + lane) * W + (k0 >> 5) + qd];
    };
    uint32_t kw0 = kword(wg, 0), kw1 = kword(wg, 1);
    for (int it = wg; it < nq; it += 2) {
      const int sb = wg, qs = it % NS;
      const int qb = q_start + it * 64;
      const uint32_t kt0 = (KT || !drop_on) ? kw0 : warp_transpose32(kw0, lane);
      const uint32_t kt1 = (KT || !drop_on) ? kw1 : warp_transpose32(kw1, lane);
      kw0 = kword(it + 2, 0);
      kw1 = kword(it + 2, 1);
      const float* stt = reinterpret_cast<const float*>(smem + C::ST_OFF + qs * 512);
      mbar_wait(&qd_full[qs], (it / NS) & 1);  // the stage's stats landed
      mbar_wait(&sd_full[sb], (it >> 1) & 1);
      // tile it-2's MMAs complete: this parity's dSᵀ buffer and the P̃ᵀ columns of its Sᵀ
      // buffer are free
      mbar_wait(&w_free[sb], ((it >> 1) & 1) ^ 1);
      const bool trw = lane == 0 && qd == 0;
      if (trw) TRACE(5, it);
      tc_fence_after();
      const bool full = !(CAUSAL && k0 + 127 > qb);
      uint8_t* drow = smem + C::DS_OFF + sb * C::DS_BYTES + row * 128;
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        uint32_t rs[32], rp[32];
        if constexpr (!STORED) tmem_ld32_nw(tl + C::S_COL + sb * 64 + h * 32, rs);
        tmem_ld32_nw(tl + C::DP_COL + sb * 64 + h * 32, rp);
        tmem_wait();
        if (trw) TRACE(h ? 8 : 6, it);
        if (h == 1) {  // both halves of Sᵀ/dPᵀ are in registers (P̃ᵀ still goes to TMEM below)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sd_free[sb]);
        }
        const uint32_t kt = h ? kt1 : kt0;
        const uint32_t sth_s = smem_u32(stt + 32 * h);
        const int q0h = qb + 32 * h;
        uint32_t pw[16], dw[16];
        auto pd_loop = [&](auto masked) {
          constexpr bool kMasked = decltype(masked)::value;
          const uint64_t sl2x2 = f32x2(sl2, sl2);
          uint32_t l4[4], d4[4];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            if ((i & 3) == 0) {  // 4 queries' statistics per 16-byte shared load (broadcast)
              asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(l4[0]), "=r"(l4[1]), "=r"(l4[2]), "=r"(l4[3]) : "r"(sth_s + 4 * i));
              asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(d4[0]), "=r"(d4[1]), "=r"(d4[2]), "=r"(d4[3]) : "r"(sth_s + 256 + 4 * i));
            }
            const uint64_t nl2 = ((uint64_t)l4[(i & 3) + 1] << 32) | l4[i & 3];
            const uint64_t nd2 = ((uint64_t)d4[(i & 3) + 1] << 32) | d4[i & 3];
            float p0, p1;
            bool k0b, k1b;
            if constexpr (STORED) {  // [64 q][128 k] tiles: query 32h + i, this thread's key
              const bf16* Pt = reinterpret_cast<const bf16*>(smem + C::PM_OFF + qs * C::PM_STAGE);
              const uint8_t* Mt = smem + C::PM_OFF + qs * C::PM_STAGE + C::P_TILE;
              const int qi = 32 * h + i;
              p0 = __bfloat162float(Pt[qi * 128 + row]);
              p1 = __bfloat162float(Pt[(qi + 1) * 128 + row]);
              k0b = Mt[qi * 128 + row] != 0;
              k1b = Mt[(qi + 1) * 128 + row] != 0;
              (void)nl2;
              (void)sl2x2;
            } else {
              float s0, s1;
              f32x2_split(ffma2(f32x2(__uint_as_float(rs[i]), __uint_as_float(rs[i + 1])), sl2x2, nl2),
                          s0, s1);
              p0 = ex2(s0);
              p1 = ex2(s1);
              k0b = (kt >> i) & 1u;
              k1b = (kt >> (i + 1)) & 1u;
            }
            if constexpr (kMasked) {
              const bool v0 = !(CAUSAL && key > q0h + i);
              const bool v1 = !(CAUSAL && key > q0h + i + 1);
              p0 = v0 ? p0 : 0.f;
              p1 = v1 ? p1 : 0.f;
              k0b = k0b && v0;
              k1b = k1b && v1;
            }
            const uint64_t kf2 = f32x2(k0b ? inv_keep : 0.f, k1b ? inv_keep : 0.f);
            const uint64_t p2 = f32x2(p0, p1);
            float a0, a1, b0, b1;
            f32x2_split(fmul2(p2, kf2), a0, a1);
            f32x2_split(
                fmul2(p2, ffma2(f32x2(__uint_as_float(rp[i]), __uint_as_float(rp[i + 1])), kf2, nd2)),
                b0, b1);
            pw[i >> 1] = pack_bf16(a0, a1);
            dw[i >> 1] = pack_bf16(b0, b1);
          }
        };
        if (full) pd_loop(std::false_type{});
        else pd_loop(std::true_type{});
        if (trw && h == 0) TRACE(7, it);
        // P̃ᵀ / dSᵀ as bf16 pairs over the first 16 of this half's (consumed) 32 Sᵀ / dPᵀ
        // columns (A operands of the TS-form dV / dK MMAs)
        tmem_st16u(tl + C::S_COL + sb * 64 + h * 32, pw);
        tmem_st16u(tl + C::DP_COL + sb * 64 + h * 32, dw);
        // dSᵀ -> smem [128 keys x 64 queries] K-major SW128: half h's queries = chunks 4h..4h+3
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int phys = (4 * h + u) ^ (row & 7);
          *reinterpret_cast<uint4*>(drow + phys * 16) =
              make_uint4(dw[4 * u], dw[4 * u + 1], dw[4 * u + 2], dw[4 * u + 3]);
        }
      }
      fence_proxy_async();
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&w_full[sb]);
      if (trw) TRACE(9, it);
    }
    // epilogue: dK·scale, dV -> bf16 (the warpgroups take alternate 32-column chunks). Rows of
    // consecutive keys are b·ld elements apart, so each warp stages its 32 rows in the K / V
    // tiles' shared memory (free: every MMA completed before acc_full; 16-byte chunks XOR-
    // swizzled by row) and stores them as row-contiguous runs instead of one 16-byte piece
    // per lane and instruction.
    mbar_wait(acc_full, 0);
    tc_fence_after();
    constexpr int ORS = HD <= 64 ? 128 : 256;  // staging row stride (bytes)
    static_assert(C::T128 >= 128 * ORS, "epilogue staging");
    uint8_t* kst = smem + C::K_OFF + qd * 32 * ORS;
    uint8_t* vst = smem + C::V_OFF + qd * 32 * ORS;
#pragma unroll 1
    for (int c = wg; c < HD / 32; c += 2) {
      float v[32], w[32];
      tmem_ld32(tl + C::DK_COL + c * 32, v);
      tmem_ld32(tl + C::DV_COL + c * 32, w);
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        const int off = lane * ORS + (((c * 32 + i) / 8) ^ (lane & 7)) * 16;
        *reinterpret_cast<uint4*>(kst + off) = make_uint4(
            pack_bf16(v[i] * a.scale, v[i + 1] * a.scale), pack_bf16(v[i + 2] * a.scale, v[i + 3] * a.scale),
            pack_bf16(v[i + 4] * a.scale, v[i + 5] * a.scale), pack_bf16(v[i + 6] * a.scale, v[i + 7] * a.scale));
        *reinterpret_cast<uint4*>(vst + off) =
            make_uint4(pack_bf16(w[i], w[i + 1]), pack_bf16(w[i + 2], w[i + 3]),
                       pack_bf16(w[i + 4], w[i + 5]), pack_bf16(w[i + 6], w[i + 7]));
      }
    }
    __syncwarp();
    const int nck = ((HD / 32 - wg + 1) / 2) * 4;  // this warpgroup's 16-byte chunks per row
    bf16* kbase = dqkv + ((int64_t)(k0 + qd * 32) * a.b + bj) * a.ld;
#pragma unroll 1
    for (int idx = lane; idx < 32 * nck; idx += 32) {
      const int r = idx / nck, k = idx % nck;
      const int ch = 4 * (wg + 2 * (k >> 2)) + (k & 3);
      const int so = r * ORS + ((ch ^ (r & 7)) * 16);
      bf16* rp = kbase + (int64_t)r * a.b * a.ld + ch * 8;
      *reinterpret_cast<uint4*>(rp + kcol) = *reinterpret_cast<const uint4*>(kst + so);
      *reinterpret_cast<uint4*>(rp + vcol) = *reinterpret_cast<const uint4*>(vst + so);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, 512);
  }
}

// -lse·log2(e) and -rowdot(dO, O) per (head, batch, query) row, and the dQ accumulator rows
// zeroed. Rows in memory order of dO / O (token-major), 4 lanes per row (as fa_delta).
template <int HD>
__global__ void fa_bwd_prep(AttnArgs a, const bf16* __restrict__ dout) {
  constexpr int VPL = HD / 32;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = t >> 2;
  const int sub = (int)(t & 3);
  const int64_t nrows = a.lh * a.b * a.s;
  const int64_t hl = r % a.lh, tok = r / a.lh;  // tok = i*b + bj
  const bf16* o = static_cast<const bf16*>(a.o);
  float acc = 0.f;
  const int64_t bj = tok % a.b, i = tok / a.b;
  const int64_t row = (hl * a.b + bj) * a.s + i;
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
      float4* z = reinterpret_cast<float4*>(a.dq_acc + row * HD + c);
      z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  if (sub == 0 && r < nrows) {
    a.bstat[row] = a.lse != nullptr ? -a.lse[row] * kLog2e : 0.f;  // (unused when STORED)
    a.bstat[nrows + row] = -acc;
  }
}

// dq_acc·scale -> bf16 into the Q columns of dqkv; rows in dqkv memory order, 8 head_dim
// elements (two float4 loads, one 16-byte store) per thread.
template <int HD>
__global__ void fa_bwd_dq_store(AttnArgs a, bf16* __restrict__ dqkv) {
  constexpr int VPR = HD / 8;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = t / VPR;
  const int v = (int)(t % VPR);
  const int64_t nrows = a.lh * a.b * a.s;
  if (r >= nrows) return;
  const int64_t hl = r % a.lh, tok = r / a.lh;
  const int64_t bj = tok % a.b, i = tok / a.b;
  const float4* src = reinterpret_cast<const float4*>(a.dq_acc + ((hl * a.b + bj) * a.s + i) * HD + v * 8);
  const float4 x = src[0], y = src[1];
  const float sc = a.scale;
  *reinterpret_cast<uint4*>(dqkv + tok * a.ld + a.qoff + hl * HD + v * 8) =
      make_uint4(pack_bf16(x.x * sc, x.y * sc), pack_bf16(x.z * sc, x.w * sc),
                 pack_bf16(y.x * sc, y.y * sc), pack_bf16(y.z * sc, y.w * sc));
}

template <int HD, bool CAUSAL, bool KT, bool STORED>
void launch_fused(const AttnArgs& a, const bf16* dout, bf16* dqkv, cudaStream_t st) {
  using C = FusedCfg<HD, STORED>;
  static_assert(C::SMEM <= 232448, "fused attention backward: smem over the limit");
  static bool once = [] {
    SPL_CUDA(cudaFuncSetAttribute(fa_bwd_fused_umma<HD, CAUSAL, KT, STORED>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    return true;
  }();
  (void)once;
  const int64_t rows = a.lh * a.b * a.s;
  fa_bwd_prep<HD><<<(unsigned)((rows * 4 + 255) / 256), 256, 0, st>>>(a, dout);
  SPL_CHECK_LAUNCH();
  const CUtensorMap m128 = attn_seq_map(a.qkv, a.ld, a.b, a.s, a.ld, 128);
  const CUtensorMap m64 = attn_seq_map(a.qkv, a.ld, a.b, a.s, a.ld, 64);
  const CUtensorMap d64 = attn_seq_map(dout, a.ldo, a.b, a.s, a.ldo, 64);
  CUtensorMap msm = m128, mmk = m128;  // unused unless STORED
  if (STORED) {
    msm = interior_map(a.sm, false, a.s, a.lh * a.b, 128, 64, false);
    mmk = interior_map(a.mask, true, a.s, a.lh * a.b, 128, 64, false);
  }
  dim3 grid((unsigned)(a.s / 128), (unsigned)(a.lh * a.b));
  static unsigned long long* trace = [] {
    const char* e = std::getenv("SPL_ATTN_TRACE");
    unsigned long long* p = nullptr;
    if (e != nullptr && e[0] == '1') {
      SPL_CUDA(cudaMalloc(&p, 16 * 64 * 8));
      SPL_CUDA(cudaMemset(p, 0, 16 * 64 * 8));
      SPL_CUDA(cudaMemcpyToSymbol(g_trace, &p, sizeof p));
    }
    return p;
  }();
  fa_bwd_fused_umma<HD, CAUSAL, KT, STORED><<<grid, 512, C::SMEM, st>>>(m128, m64, d64, msm, mmk, a, dqkv);
  SPL_CHECK_LAUNCH();
  static int traced = 0;
  if (trace != nullptr && traced++ == 2 && grid.x > kTraceX && grid.y > kTraceY) {
    unsigned long long h[16 * 64];
    SPL_CUDA(cudaStreamSynchronize(st));
    SPL_CUDA(cudaMemcpy(h, trace, sizeof h, cudaMemcpyDeviceToHost));
    const unsigned long long t0 = h[15 * 64];
    fprintf(stderr, "fused bwd trace (cycles from CTA start), columns: tile, mma[issue_sd wait-start, "
                    "sd issued, w_full seen, dq_free seen, end], sm[ready, ld0, cmp0, ld1, w_full], "
                    "rd[dq_full, ld, reds], tma[empty]\n");
    for (int it = 0; it < 32; ++it) {
      fprintf(stderr, "%2d", it);
      for (int e : {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13})
        fprintf(stderr, " %7lld", h[e * 64 + it] ? (long long)(h[e * 64 + it] - t0) : -1ll);
      fprintf(stderr, "\n");
    }
  }
  fa_bwd_dq_store<HD><<<(unsigned)((rows * (HD / 8) + 255) / 256), 256, 0, st>>>(a, dqkv);
  SPL_CHECK_LAUNCH();
}

}  // namespace

bool attn_bwd_fused_supported(const AttnArgs& a) {
  static const bool off = [] {
    const char* e = std::getenv("SPL_ATTN_DETERMINISTIC");
    return e != nullptr && e[0] == '1';
  }();
  const bool regime_ok = a.sm == nullptr
                             ? (a.lse != nullptr && (a.keepbits != nullptr || a.drop.thresh == 0))
                             : (a.mask != nullptr && ((uintptr_t)a.sm & 15) == 0 &&
                                ((uintptr_t)a.mask & 15) == 0);
  return !off && regime_ok && a.dq_acc != nullptr && a.bstat != nullptr &&
         (a.hd == 64 || a.hd == 96) && a.s % 128 == 0 && a.s >= 128 && a.ld % 8 == 0 && a.ldo % 8 == 0 &&
         a.qoff % 8 == 0 && ((uintptr_t)a.qkv & 15) == 0 && ((uintptr_t)a.o & 15) == 0 &&
         ((uintptr_t)a.dq_acc & 15) == 0 && ((uintptr_t)a.bstat & 15) == 0 && a.s < (1 << 30);
}

void attn_bwd_fused(const AttnArgs& a, const void* dout, void* dqkv, cudaStream_t st) {
  const bf16* d = static_cast<const bf16*>(dout);
  bf16* g = static_cast<bf16*>(dqkv);
#define SPL_FUSED_CASE(HDX)                                                              \
  if (a.sm != nullptr) {                                                                 \
    if (a.causal) launch_fused<HDX, true, false, true>(a, d, g, st);                     \
    else launch_fused<HDX, false, false, true>(a, d, g, st);                             \
  } else if (a.keep_t) {                                                                 \
    if (a.causal) launch_fused<HDX, true, true, false>(a, d, g, st);                     \
    else launch_fused<HDX, false, true, false>(a, d, g, st);                             \
  } else {                                                                               \
    if (a.causal) launch_fused<HDX, true, false, false>(a, d, g, st);                    \
    else launch_fused<HDX, false, false, false>(a, d, g, st);                            \
  }
  if (a.hd == 64) {
    SPL_FUSED_CASE(64)
  } else {
    SPL_FUSED_CASE(96)
  }
#undef SPL_FUSED_CASE
}

}  // namespace spl::k
