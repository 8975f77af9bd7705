// Attention forward on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), bf16, for the
// selective-recompute regime: stores only O and the row LSE.
//
// CTA = 128 queries of one (head, batch). Warp roles (320 threads):
//   warp 0      TMA producer: Q once, then K (pass 1) / K,V (pass 2) 128-key tiles, 2 stages
//   warp 1      TMEM allocator + single-thread MMA issuer
//   warps 2..9  softmax: query row = TMEM lane (warp w reads lanes 32*(w%4)..); warps 2-5 take
//               keys 0-63 of each tile, warps 6-9 keys 64-127 (row statistics merged via smem)
// Selective / full regimes: ONE pass over the keys with a lazily rescaled O (online softmax):
//   S = Q·Kᵀ -> row max over both column halves (exchanged through smem per tile); the
//   reference point m_used moves only when the max grows by more than 2^8, and then O (TMEM)
//   and l are rescaled once PV of the previous tile has completed (rare after the first tile);
//   P̃ = exp2(S·c - m_used)·keep (≤ 2^8, bf16) -> smem (UMMA K-major SW128) -> O += P̃·V;
//   epilogue O · (1/(1-p))/l, LSE = m_used + log2 l.
// No-recompute regime (MAT): two passes (pass 1 row max/sum, pass 2 normalised P), because the
//   stored softmax_out must be normalised when it is written.
// TMEM: S double-buffered (2 × 128 fp32 columns) + O (HD columns). MMAs of tile j+1 overlap
// the softmax of tile j. SMEM: Q 32 KB, 2 × (K, V) 128 KB, 2 × P 64 KB.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace spl::k {

namespace {

using namespace tc;

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kAtomBytes = 128 * 128;  // 128 rows x 128 B (64 bf16) swizzle-128B atom block

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int HD, bool PT>
struct FwdCfg {
  static constexpr int ATOMS = (HD + 63) / 64;
  static constexpr int TILE = ATOMS * kAtomBytes;  // one 128-row tile of Q, K or V
  // K/V ring depth: head_dim <= 128 takes 2 stages, or 3 when P̃ lives in TMEM (PT) and its
  // 64 KB of smem are free; head_dim 160 (3 atoms, 48 KB tiles) fits one.
  static constexpr int KVS = HD > 128 ? 1 : (PT ? 3 : 2);
  static constexpr int Q_OFF = 0;
  static constexpr int KV_OFF = TILE;                   // [KVS stages][K tile, V tile]
  static constexpr int P_OFF = KV_OFF + KVS * 2 * TILE; // [2][128 x 128 bf16] (!PT)
  static constexpr int P_BYTES = 2 * kAtomBytes;
  static constexpr int BAR_OFF = P_OFF + (PT ? 0 : 2 * P_BYTES);
  // [2 halves][128 rows] (m, l) exchanged between pass 1 and pass 2, when the P buffers are
  // not in use yet (smem is at the 227 KB limit for HD = 96/128)
  static constexpr int STAT_OFF = P_OFF;
  static_assert(STAT_OFF % 1024 == 0, "stats exchange area alignment");
  static constexpr int XCH_OFF = BAR_OFF + 256;  // [2 halves][128 rows] floats (single pass)
  static constexpr int SMEM = XCH_OFF + 1024 + 1024;
  static constexpr int O_COL = 256;  // O accumulator columns [256, 256 + HD)
};

// MAT (no-recompute regime): pass 2 also writes the interior the reference stores —
// softmax_out P, the softmax-dropout mask (the raw keep bit at every position, block.cpp:
// 392-394) and softmax_dropout_out P·mask/(1-p) — as {lh, b, s, s} rows (bf16, u8, bf16);
// every key tile is visited (causal-masked tiles still carry mask bits).
// PT (single pass only): P̃ goes to TMEM (over the consumed half of its S buffer) and the
// P̃·V MMA reads A from TMEM, instead of a swizzled smem tile + proxy fence.
template <int HD, bool CAUSAL, bool MAT, bool PT>
__global__ void __launch_bounds__(320, 1)
    fa_fwd_umma(const __grid_constant__ CUtensorMap map_qkv, AttnArgs a) {
  using Cfg = FwdCfg<HD, PT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* Qs = smem + Cfg::Q_OFF;
  uint8_t* KVs = smem + Cfg::KV_OFF;
  uint8_t* Ps = smem + Cfg::P_OFF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;   // [3] (KVS used)
  uint64_t* kv_empty = bar + 4;  // [3]
  uint64_t* s_full = bar + 7;    // [2]
  uint64_t* s_free = bar + 9;    // [2]
  uint64_t* p_full = bar + 11;   // [2]
  uint64_t* p_free = bar + 13;   // [2]
  uint64_t* o_full = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);
  uint64_t* o_done = bar + 17;   // one phase per P̃·V MMA (single pass: gates O rescaling)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * 128;
  const int hl = blockIdx.y / (int)a.b, bj = blockIdx.y % (int)a.b;
  const int S = (int)a.s;
  const int kv_end = (CAUSAL && !MAT) ? min(S, q0 + 128) : S;
  const int nkv = (kv_end + 127) / 128;
  const int qcol = (int)(a.qoff + (int64_t)hl * HD), kcol = (int)(a.koff + (int64_t)hl * HD),
            vcol = (int)(a.voff + (int64_t)hl * HD);

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < Cfg::KVS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&p_free[i], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_qkv) : "memory");
  }
  if (warp == 1) tmem_alloc_warp(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      mbar_expect_tx(q_full, Cfg::TILE);
#pragma unroll
      for (int at = 0; at < Cfg::ATOMS; ++at)
        tma_load_3d(Qs + at * kAtomBytes, &map_qkv, q_full, qcol + 64 * at, bj, q0);
      int it = 0;
      constexpr int PASSES = MAT ? 2 : 1;
      for (int pass = 0; pass < PASSES; ++pass) {
        const bool with_v = pass == PASSES - 1;
        for (int j = 0; j < nkv; ++j, ++it) {
          const int st = it % Cfg::KVS;
          mbar_wait(&kv_empty[st], ((it / Cfg::KVS) & 1) ^ 1);
          uint8_t* Kt = KVs + st * 2 * Cfg::TILE;
          uint8_t* Vt = Kt + Cfg::TILE;
          mbar_expect_tx(&kv_full[st], (with_v ? 2 : 1) * Cfg::TILE);
#pragma unroll
          for (int at = 0; at < Cfg::ATOMS; ++at)
            tma_load_3d(Kt + at * kAtomBytes, &map_qkv, &kv_full[st], kcol + 64 * at, bj, j * 128);
          if (with_v) {
#pragma unroll
            for (int at = 0; at < Cfg::ATOMS; ++at)
              tma_load_3d(Vt + at * kAtomBytes, &map_qkv, &kv_full[st], vcol + 64 * at, bj, j * 128);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = make_idesc(128, 128, false, false);
      constexpr uint32_t idesc_o = make_idesc(128, HD, false, true);
      const uint32_t qa = smem_u32(Qs);
      mbar_wait(q_full, 0);
      int it = 0, sc = 0;
      auto issue_s = [&](int stage_it) {  // S[sc%2] = Q · K(stage)ᵀ
        const int st = stage_it % Cfg::KVS;
        mbar_wait(&kv_full[st], (stage_it / Cfg::KVS) & 1);
        const int sb = sc & 1;
        mbar_wait(&s_free[sb], ((sc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t kb = smem_u32(KVs + st * 2 * Cfg::TILE);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtomBytes + (kk & 3) * 32;
          umma_bf16(tmem + sb * 128, desc_add(smem_desc(qa, 16, 1024), off >> 4), desc_add(smem_desc(kb, 16, 1024), off >> 4),
                    idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[sb]);
        ++sc;
      };
      if constexpr (MAT) {  // pass 1 (statistics only)
        for (int j = 0; j < nkv; ++j, ++it) {
          issue_s(it);
          umma_commit(&kv_empty[it % Cfg::KVS]);
        }
      }
      // pass 2: S_{j+1} is issued before PV_j so the softmax of j+1 can start early — unless
      // the K/V ring has one stage (head_dim 160), where K_{j+1} can only arrive after PV_j
      // has released the stage
      constexpr bool kAhead = Cfg::KVS > 1;
      const int base = it;
      issue_s(base);
      for (int j = 0; j < nkv; ++j) {
        if (kAhead && j + 1 < nkv) issue_s(base + j + 1);
        const int pb = j & 1;
        mbar_wait(&p_full[pb], (j >> 1) & 1);
        tc_fence_after();
        const int st = (base + j) % Cfg::KVS;
        const uint32_t pa = smem_u32(Ps + pb * Cfg::P_BYTES);
        const uint32_t vb = smem_u32(KVs + st * 2 * Cfg::TILE + Cfg::TILE);
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk) {
          const uint64_t bd = desc_add(smem_desc(vb, kAtomBytes, 1024), kk * (2048 >> 4));
          if constexpr (PT) {  // P̃ of tile j over the first 64 columns of its S buffer
            const uint32_t ta = tmem + (uint32_t)(((base + j) & 1) * 128 + kk * 8);
            umma_bf16_ts(tmem + Cfg::O_COL, ta, bd, idesc_o, (j | kk) != 0 ? 1u : 0u);
          } else {
            const uint64_t ad = desc_add(smem_desc(pa, 16, 1024), ((kk >> 2) * kAtomBytes + (kk & 3) * 32) >> 4);
            umma_bf16(tmem + Cfg::O_COL, ad, bd, idesc_o, (j | kk) != 0 ? 1u : 0u);
          }
        }
        umma_commit(&p_free[pb]);
        umma_commit(&kv_empty[st]);
        umma_commit(o_done);
        if (!kAhead && j + 1 < nkv) issue_s(base + j + 1);
      }
      umma_commit(o_full);
    }
  } else {
    // ------------------------------------------------ softmax warps
    const int qd = warp & 3;
    const int half = (warp - 2) >> 2;  // 0: keys 0-63 of a tile, 1: keys 64-127
    const int row = qd * 32 + lane;
    const int qr = q0 + row;
    const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);
    const float sl2 = a.scale * kLog2e;
    const bool drop_on = a.drop.thresh != 0;
    const int W = (S + 31) / 32;
    const int64_t brow = ((int64_t)hl * a.b + bj) * a.s;
    const uint32_t* kbits = a.keepbits + (brow + (qr < S ? qr : 0)) * W;
    float m, l;
    float oscale = 1.f;
    if constexpr (MAT) {
      float2* stat = reinterpret_cast<float2*>(smem + Cfg::STAT_OFF);
      m = -INFINITY;
      l = 0.f;
      int sc = 0;
      // a tile needs per-element masking only at the sequence tail or on the causal diagonal
      auto tile_full = [&](int j) {
        return j * 128 + 128 <= S && !(CAUSAL && j * 128 + 127 > q0);
      };
      // pass 1: statistics of this half's 64 columns
      for (int j = 0; j < nkv; ++j, ++sc) {
        const int sb = sc & 1;
        mbar_wait(&s_full[sb], (sc >> 1) & 1);
        tc_fence_after();
        uint32_t r0[32], r1[32];
        tmem_ld32_nw(tl + sb * 128 + half * 64, r0);
        tmem_ld32_nw(tl + sb * 128 + half * 64 + 32, r1);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[sb]);  // S buffer may be overwritten now
        float v[64];
  #pragma unroll
        for (int i = 0; i < 32; ++i) {
          v[i] = __uint_as_float(r0[i]) * sl2;
          v[32 + i] = __uint_as_float(r1[i]) * sl2;
        }
        if (!tile_full(j)) {
          const int k0 = j * 128 + half * 64;
  #pragma unroll
          for (int i = 0; i < 64; ++i)
            if (k0 + i >= S || (CAUSAL && k0 + i > qr)) v[i] = -INFINITY;
        }
        float cm = v[0];
  #pragma unroll
        for (int i = 1; i < 64; ++i) cm = fmaxf(cm, v[i]);
        const float mn = fmaxf(m, cm);
        if (mn != -INFINITY) {
          float sum = 0.f;
  #pragma unroll
          for (int i = 0; i < 64; ++i) sum += ex2(v[i] - mn);
          l = l * ex2(m - mn) + sum;
          m = mn;
        }
      }
      // merge the two halves' (m, l) of each row
      stat[half * 128 + row] = make_float2(m, l);
      asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 softmax warps only
      {
        const float2 o = stat[(half ^ 1) * 128 + row];
        const float mn = fmaxf(m, o.x);
        if (mn != -INFINITY) {
          l = (m == -INFINITY ? 0.f : l * ex2(m - mn)) + (o.x == -INFINITY ? 0.f : o.y * ex2(o.x - mn));
          m = mn;
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");  // stats read before P overwrites them
      const float scale_p = a.drop.inv_keep / l;  // 1/l and the dropout rescale folded
      const float inv_l = 1.0f / l;
      const float mm = m == -INFINITY ? 0.f : m;
      // pass 2: probabilities -> P̃ (bf16, K-major SW128 in smem)
      const int kw0 = half * 2;  // this half's first 32-key word within a tile
      uint2 wnext = make_uint2(0xffffffffu, 0xffffffffu);
      auto load_words = [&](int j) {
        uint2 w = make_uint2(0xffffffffu, 0xffffffffu);
        if (drop_on) {
          const int wd = j * 4 + kw0;
          w.x = (qr < S && wd < W) ? kbits[wd] : 0u;
          w.y = (qr < S && wd + 1 < W) ? kbits[wd + 1] : 0u;
        }
        return w;
      };
      if (nkv > 0) wnext = load_words(0);
      for (int j = 0; j < nkv; ++j, ++sc) {
        const int sb = sc & 1, pb = j & 1;
        const uint2 wcur = wnext;
        if (j + 1 < nkv) wnext = load_words(j + 1);  // prefetch the next tile's keep bits
        mbar_wait(&s_full[sb], (sc >> 1) & 1);
        tc_fence_after();
        uint32_t r0[32], r1[32];
        tmem_ld32_nw(tl + sb * 128 + half * 64, r0);
        tmem_ld32_nw(tl + sb * 128 + half * 64 + 32, r1);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[sb]);
        mbar_wait(&p_free[pb], ((j >> 1) & 1) ^ 1);
        const bool full = tile_full(j);
        const int k0 = j * 128 + half * 64;
        uint32_t pk[32];
        uint32_t pm[MAT ? 32 : 1];  // MAT: softmax_out pairs
  #pragma unroll
        for (int i = 0; i < 64; i += 2) {
          float p2[2], pn[2];
  #pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int e = i + u;
            const float sv = __uint_as_float(e < 32 ? r0[e] : r1[e - 32]);
            const uint32_t word = e < 32 ? wcur.x : wcur.y;
            const bool keep = (word >> (e & 31)) & 1u;
            float p;
            if constexpr (MAT) {
              pn[u] = ex2(sv * sl2 - mm) * inv_l;
              if (!full && (k0 + e >= S || (CAUSAL && k0 + e > qr))) pn[u] = 0.f;
              p = pn[u] * a.drop.inv_keep;
            } else {
              p = ex2(sv * sl2 - mm) * scale_p;
              if (!full && (k0 + e >= S || (CAUSAL && k0 + e > qr))) p = 0.f;
            }
            p2[u] = keep ? p : 0.f;
          }
          pk[i >> 1] = pack_bf16(p2[0], p2[1]);
          if constexpr (MAT) pm[i >> 1] = pack_bf16(pn[0], pn[1]);
        }
        if constexpr (MAT) {  // S % 64 == 0 (dispatcher): a half-tile is all in or all out
          if (qr < S && k0 < S) {
            const int64_t mi = (brow + qr) * (int64_t)S + k0;
            uint8_t* smo = reinterpret_cast<uint8_t*>(static_cast<bf16*>(a.sm) + mi);
            uint8_t* sdo = reinterpret_cast<uint8_t*>(static_cast<bf16*>(a.sd) + mi);
            uint8_t* mko = a.mask + mi;
  #pragma unroll
            for (int u = 0; u < 4; ++u) {
              st_v8(smo + 32 * u, pm[8 * u], pm[8 * u + 1], pm[8 * u + 2], pm[8 * u + 3], pm[8 * u + 4],
                    pm[8 * u + 5], pm[8 * u + 6], pm[8 * u + 7]);
              st_v8(sdo + 32 * u, pk[8 * u], pk[8 * u + 1], pk[8 * u + 2], pk[8 * u + 3], pk[8 * u + 4],
                    pk[8 * u + 5], pk[8 * u + 6], pk[8 * u + 7]);
            }
            const uint32_t wb[2] = {wcur.x, wcur.y};
  #pragma unroll
            for (int u = 0; u < 2; ++u) {  // 32 keys -> 32 mask bytes
              uint32_t q8[8];
  #pragma unroll
              for (int v = 0; v < 8; ++v) {
                const uint32_t bits = (wb[u] >> (4 * v)) & 0xFu;
                q8[v] = (bits & 1u) | ((bits & 2u) << 7) | ((bits & 4u) << 14) | ((bits & 8u) << 21);
              }
              st_v8(mko + 32 * u, q8[0], q8[1], q8[2], q8[3], q8[4], q8[5], q8[6], q8[7]);
            }
          }
        }
        uint8_t* prow = Ps + pb * Cfg::P_BYTES + row * 128;
        // this half's keys = logical 16 B chunks 8*half .. 8*half+7 = atom `half`, swizzled by row
  #pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int phys = u ^ (row & 7);
          *reinterpret_cast<uint4*>(prow + half * kAtomBytes + phys * 16) =
              make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb]);
      }

    } else {
      float m_used = -INFINITY;
      l = 0.f;
      int sc = 0;
      auto tile_full = [&](int j) {
        return j * 128 + 128 <= S && !(CAUSAL && j * 128 + 127 > q0);
      };
      float* xch = reinterpret_cast<float*>(smem + Cfg::XCH_OFF);  // [half][row]
      const int kw0 = half * 2;  // this half's first 32-key word within a tile
      auto load_words = [&](int j) {
        uint2 w = make_uint2(0xffffffffu, 0xffffffffu);
        if (drop_on) {
          const int wd = j * 4 + kw0;
          w.x = (qr < S && wd < W) ? kbits[wd] : 0u;
          w.y = (qr < S && wd + 1 < W) ? kbits[wd + 1] : 0u;
        }
        return w;
      };
      auto pair_sync = [&] { asm volatile("bar.sync %0, 64;" ::"r"(2 + qd) : "memory"); };
      // keep-bit words two tiles ahead (the loads miss L2 and were waited on one tile ahead)
      uint2 wnext = nkv > 0 ? load_words(0) : make_uint2(0u, 0u);
      uint2 wnext2 = nkv > 1 ? load_words(1) : make_uint2(0u, 0u);
      for (int j = 0; j < nkv; ++j, ++sc) {
        const int sb = sc & 1, pb = j & 1;
        const uint2 wcur = wnext;
        wnext = wnext2;
        if (j + 2 < nkv) wnext2 = load_words(j + 2);
        mbar_wait(&s_full[sb], (sc >> 1) & 1);
        tc_fence_after();
        uint32_t r0[32], r1[32];
        tmem_ld32_nw(tl + sb * 128 + half * 64, r0);
        tmem_ld32_nw(tl + sb * 128 + half * 64 + 32, r1);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[sb]);
        const bool full = tile_full(j);
        const int k0 = j * 128 + half * 64;
        float v[64];
        {  // scores · scale·log2e in packed fp32x2 multiplies (bit-identical to the scalar form)
          const uint64_t sl2x2 = f32x2(sl2, sl2);
  #pragma unroll
          for (int i = 0; i < 32; i += 2) {
            f32x2_split(fmul2(f32x2(__uint_as_float(r0[i]), __uint_as_float(r0[i + 1])), sl2x2),
                        v[i], v[i + 1]);
            f32x2_split(fmul2(f32x2(__uint_as_float(r1[i]), __uint_as_float(r1[i + 1])), sl2x2),
                        v[32 + i], v[32 + i + 1]);
          }
        }
        if (!full) {
  #pragma unroll
          for (int i = 0; i < 64; ++i)
            if (k0 + i >= S || (CAUSAL && k0 + i > qr)) v[i] = -INFINITY;
        }
        float cm = v[0];
  #pragma unroll
        for (int i = 1; i < 64; ++i) cm = fmaxf(cm, v[i]);
        // row max of the whole tile: exchange with the partner warp (same rows, other half)
        xch[half * 128 + row] = cm;
        pair_sync();
        const float mt = fmaxf(cm, xch[(half ^ 1) * 128 + row]);
        pair_sync();  // both read before the next tile's write
        bool rescale = false;
        float f = 1.f;
        if (m_used == -INFINITY) {
          m_used = mt;  // O and l are still zero: nothing to rescale
        } else if (mt > m_used + 8.f) {
          f = ex2(m_used - mt);
          m_used = mt;
          l *= f;
          rescale = true;
        }
        const float mm = m_used == -INFINITY ? 0.f : m_used;
        mbar_wait(&p_free[pb], ((j >> 1) & 1) ^ 1);
        if (__any_sync(0xffffffffu, rescale)) {
          // O += P̃·V of tile j-1 must have landed before O is rescaled in TMEM
          mbar_wait(o_done, (j - 1) & 1);
          tc_fence_after();
  #pragma unroll 1
          for (int c = half; c < HD / 32; c += 2) {
            float o[32];
            tmem_ld32(tl + Cfg::O_COL + c * 32, o);
  #pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= f;
            tmem_st32(tl + Cfg::O_COL + c * 32, o);
          }
        }
        uint32_t pk[32];
        float ls = 0.f;
        const uint64_t nmm2 = f32x2(-mm, -mm);
  #pragma unroll
        for (int i = 0; i < 64; i += 2) {
          float x[2], p2[2];
          f32x2_split(fadd2(f32x2(v[i], v[i + 1]), nmm2), x[0], x[1]);  // v - m, packed
  #pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int e = i + u;
            const uint32_t word = e < 32 ? wcur.x : wcur.y;
            const bool keep = (word >> (e & 31)) & 1u;
            const float p = ex2(x[u]);
            ls += p;
            p2[u] = keep ? p : 0.f;
          }
          pk[i >> 1] = pack_bf16(p2[0], p2[1]);
        }
        l += ls;
        if constexpr (PT) {
          tmem_st32u(tl + sb * 128 + half * 32, pk);  // keys 64*half.. as bf16 pairs
        } else {
          uint8_t* prow = Ps + pb * Cfg::P_BYTES + row * 128;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int phys = u ^ (row & 7);
            *reinterpret_cast<uint4*>(prow + half * kAtomBytes + phys * 16) =
                make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          }
          fence_proxy_async();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb]);
      }
      // l of the whole row: both halves share m_used
      xch[half * 128 + row] = l;
      pair_sync();
      l += xch[(half ^ 1) * 128 + row];
      m = m_used;
      oscale = a.drop.inv_keep / l;

    }
    // epilogue: O · oscale -> bf16; the halves take alternate 32-column chunks
    mbar_wait(o_full, 0);
    tc_fence_after();
    bf16* out = static_cast<bf16*>(a.o) + ((int64_t)(qr < S ? qr : 0) * a.b + bj) * a.ldo +
                (int64_t)hl * HD;
#pragma unroll 1
    for (int c = half; c < HD / 32; c += 2) {
      float v[32];
      tmem_ld32(tl + Cfg::O_COL + c * 32, v);
      if (qr < S) {
        if ((((uintptr_t)(out + c * 32)) & 31) == 0) {  // full 32-byte sectors per lane
#pragma unroll
          for (int i = 0; i < 32; i += 16)
            st_v8(out + c * 32 + i, pack_bf16(v[i] * oscale, v[i + 1] * oscale),
                  pack_bf16(v[i + 2] * oscale, v[i + 3] * oscale), pack_bf16(v[i + 4] * oscale, v[i + 5] * oscale),
                  pack_bf16(v[i + 6] * oscale, v[i + 7] * oscale), pack_bf16(v[i + 8] * oscale, v[i + 9] * oscale),
                  pack_bf16(v[i + 10] * oscale, v[i + 11] * oscale), pack_bf16(v[i + 12] * oscale, v[i + 13] * oscale),
                  pack_bf16(v[i + 14] * oscale, v[i + 15] * oscale));
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 8)
            *reinterpret_cast<uint4*>(out + c * 32 + i) =
                make_uint4(pack_bf16(v[i] * oscale, v[i + 1] * oscale),
                           pack_bf16(v[i + 2] * oscale, v[i + 3] * oscale),
                           pack_bf16(v[i + 4] * oscale, v[i + 5] * oscale),
                           pack_bf16(v[i + 6] * oscale, v[i + 7] * oscale));
        }
      }
    }
    if (half == 0 && qr < S && a.lse) a.lse[brow + qr] = (m + log2f(l)) * kLn2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, 512);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    SPL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (p == nullptr || q != cudaDriverEntryPointSuccess) raise(3, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

}  // namespace

// 3-D map over a {s, b, width} row-major bf16 buffer (row = s_i*b + b_j, stride ld elements):
// dims {width, b, s}; box {64, 1, rows}; 128 B swizzle.
CUtensorMap attn_seq_map(const void* ptr, int64_t width, int64_t b, int64_t s, int64_t ld, int rows) {
  static std::mutex mu;
  static std::unordered_map<std::string, CUtensorMap> cache;
  char key[160];
  snprintf(key, sizeof key, "%p/%lld/%lld/%lld/%lld/%d", ptr, (long long)width, (long long)b,
           (long long)s, (long long)ld, rows);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  const cuuint64_t dims[3] = {(cuuint64_t)width, (cuuint64_t)b, (cuuint64_t)s};
  const cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(b * ld * 2)};
  const cuuint32_t box[3] = {64, 1, (cuuint32_t)rows};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(3, "cuTensorMapEncodeTiled (attention) failed: " + std::to_string((int)r));
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  return m;
}

namespace {

template <int HD, bool CAUSAL, bool MAT, bool PT>
void launch_fwd_umma(const AttnArgs& a, cudaStream_t st) {
  using Cfg = FwdCfg<HD, PT>;
  static_assert(Cfg::SMEM <= 232448, "attention forward: smem over the limit");
  static bool once = [] {
    SPL_CUDA(cudaFuncSetAttribute(fa_fwd_umma<HD, CAUSAL, MAT, PT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    return true;
  }();
  (void)once;
  const CUtensorMap mq = attn_seq_map(a.qkv, a.ld, a.b, a.s, a.ld, 128);
  dim3 grid((unsigned)((a.s + 127) / 128), (unsigned)(a.lh * a.b));
  fa_fwd_umma<HD, CAUSAL, MAT, PT><<<grid, 320, Cfg::SMEM, st>>>(mq, a);
  SPL_CHECK_LAUNCH();
}
bool fwd_p_tmem() {
  static const bool on = [] {
    const char* e = std::getenv("SPL_ATTN_P_TMEM");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}
template <int HD>
void launch_fwd_umma_hd(const AttnArgs& a, cudaStream_t st) {
  if (a.sm != nullptr) {
    if (a.causal) launch_fwd_umma<HD, true, true, false>(a, st);
    else launch_fwd_umma<HD, false, true, false>(a, st);
  } else if (fwd_p_tmem()) {
    if (a.causal) launch_fwd_umma<HD, true, false, true>(a, st);
    else launch_fwd_umma<HD, false, false, true>(a, st);
  } else {
    if (a.causal) launch_fwd_umma<HD, true, false, false>(a, st);
    else launch_fwd_umma<HD, false, false, false>(a, st);
  }
}

}  // namespace

bool attn_fwd_umma_supported(const AttnArgs& a) {
  const bool hd_ok = a.hd == 64 || a.hd == 96 || a.hd == 128 || a.hd == 160;
  const bool regime_ok = a.sm == nullptr
                             ? a.lse != nullptr
                             : (a.mask != nullptr && a.sd != nullptr && a.s % 64 == 0 &&
                                ((uintptr_t)a.sm & 15) == 0 && ((uintptr_t)a.sd & 15) == 0 &&
                                ((uintptr_t)a.mask & 15) == 0);
  return hd_ok && regime_ok && a.ld % 8 == 0 && a.ldo % 8 == 0 &&
         ((uintptr_t)a.qkv & 15) == 0 && ((uintptr_t)a.o & 15) == 0 &&
         (a.keepbits != nullptr || a.drop.thresh == 0) && a.s < (1 << 30);
}

void attn_fwd_umma(const AttnArgs& a, cudaStream_t st) {
  if (attn_fwd_pp_supported(a)) return attn_fwd_pp(a, st);
  switch (a.hd) {
    case 64: return launch_fwd_umma_hd<64>(a, st);
    case 96: return launch_fwd_umma_hd<96>(a, st);
    case 128: return launch_fwd_umma_hd<128>(a, st);
    case 160: return launch_fwd_umma_hd<160>(a, st);
    default: raise(3, "attn_fwd_umma: unsupported head_dim");
  }
}

}  // namespace spl::k
