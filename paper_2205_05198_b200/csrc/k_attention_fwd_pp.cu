// Attention forward, recompute regimes (selective / full): two 128-query tiles per CTA in
// ping-pong (block.cpp:381-417 with the dropout of block.cpp:393-414; stores only O and the row
// LSE, the interior is recomputed in the backward).
//
// CTA = 256 queries (tiles 0 and 1) of one (head, batch); 384 threads:
//   warp 0      TMA producer: Q0, Q1 once, then (K, V) 128-key tiles through a KVS-stage ring
//   warp 1      TMEM allocator + MMA issuer (warp-converged, one elected lane issues)
//   warps 2, 3  idle (with warps 0, 1 they hand registers to the softmax warps: setmaxnreg)
//   warps 4-7   softmax of tile 0, warps 8-11 softmax of tile 1: one thread per query row
//               (TMEM lane), the whole 128-key row of S in registers — no cross-warp exchange.
// Per key tile j the MMA warp issues P̃0(j)·V, S0(j+1), P̃1(j)·V, S1(j+1): while warpgroup 0
// exponentiates, the tensor cores run tile 1's products and vice versa. Because S_t(j+1) is
// issued after P̃_t(j)·V, the commit that signals S_t(j+1) covers that product too, so the
// softmax may rescale O_t in TMEM as soon as it sees S_t(j+1).
// Online softmax with a lazily moved reference point (as fa_fwd_umma): m_used moves only when
// the row max grows by more than 2^8 (O and l then rescaled once); P̃ = 2^(S·c - m_used)·keep as
// bf16 pairs written back over the first 64 columns of the consumed S tile and read by a TS-form
// tcgen05.mma (O += P̃·V). Epilogue O·(1/(1-p))/l and LSE = (m_used + log2 l)·ln 2.
// TMEM (512 columns): S0 [0,128), S1 [128,256), O0 [256,256+HD), O1 [256+HD,256+2HD).
// Measured (22B, hd 96, ncu): 548 µs vs 675 µs for fa_fwd_umma. A variant with 64-key steps
// and the S columns of a tile double-buffered (so the softmax never waits for Q·Kᵀ) measured
// slower (625 µs): it issues 20 instead of 14 MMAs per 128 keys and tile, and the MMA warp's
// issue rate (≈ one tcgen05.mma per 75-100 cycles here, with the softmax warps' tcgen05.ld /
// st in flight) is what bounds both.
// Requirements (else fa_fwd_umma): head_dim 64/96/128, s % 128 == 0, keep bits in the row layout.
#include <cstdlib>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace spl::k {

CUtensorMap attn_seq_map(const void* ptr, int64_t width, int64_t b, int64_t s, int64_t ld, int rows);

namespace {

using namespace tc;

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr int kAtomBytes = 128 * 128;
constexpr int kPolyDefault = 4;  // SPL_ATTN_POLY default (see poly_period)

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for a pair of x <= 0 (or -inf) on the FMA pipe instead of the MUFU (XU) pipe, which the
// ncu capture of this kernel shows as its busiest (XU 52 % active vs FMA 17 %): x clamped to
// -126 (p < 1 has exponent field 126, so j >= -126 keeps the sum's exponent field >= 0),
// j = floor(x) by a round-down add of 1.5·2^23 (j sits in the sum's low mantissa bits),
// 2^(x-j) by a degree-3 polynomial on [0, 1) (relative error <= 8.6e-5, far below the bf16
// rounding of P̃), and j added into the exponent field: (t_bits << 23) == j << 23 (mod 2^32).
// Clamped values give a value <= 2^-125 instead of 0: below any bf16 / fp32 sum's ulp.
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x) {
  float x0, x1;
  f32x2_split(x, x0, x1);
  const uint64_t xc = f32x2(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  uint64_t t;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(t) : "l"(xc), "l"(f32x2(12582912.f, 12582912.f)));
  const uint64_t jf = fadd2(t, f32x2(-12582912.f, -12582912.f));  // exact
  const uint64_t fr = ffma2(jf, f32x2(-1.f, -1.f), xc);             // x - j in [0, 1), exact
  uint64_t p = ffma2(f32x2(0.07706602f, 0.07706602f), fr, f32x2(0.22764611f, 0.22764611f));
  p = ffma2(p, fr, f32x2(0.69511652f, 0.69511652f));
  p = ffma2(p, fr, f32x2(1.f, 1.f));  // p(0) = 1: the row maximum's exponential is exact
  float p0, p1, t0, t1;
  f32x2_split(p, p0, p1);
  f32x2_split(t, t0, t1);
  return f32x2(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(t0) << 23)),
               __uint_as_float(__float_as_uint(p1) + (__float_as_uint(t1) << 23)));
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
template <int HD>
struct PpCfg {
  static constexpr int ATOMS = (HD + 63) / 64;
  static constexpr int TILE = ATOMS * kAtomBytes;
  static constexpr int KVS = HD <= 64 ? 4 : 2;  // (K, V) ring depth, 128 keys per stage
  static constexpr int ORS = HD <= 64 ? 128 : 256;  // epilogue staging row stride (bytes)
  static_assert(TILE >= 128 * ORS && HD * 2 <= ORS, "epilogue staging: 128 rows per Q tile");
  static constexpr int KV_OFF = 2 * TILE;
  static constexpr int BAR_OFF = KV_OFF + KVS * 2 * TILE;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr int O_COL = 256;
};

// MAT (no-recompute regime): two passes over the keys — pass 1 the row max and sum (Q·Kᵀ and
// exponentials only), pass 2 the normalised P = softmax_out, the mask (the raw keep bit at every
// position, block.cpp:392-394) and P̃ = P·mask/(1-p) = softmax_dropout_out, written to the
// stored interior with 32-byte stores, and O += P̃·V (O needs no final rescale). Every key
// tile is visited, causal ones included (the stored mask carries all bits).
// PE: every PE-th element pair of the recompute loop takes its exponentials from ex2_poly2
// (0: all on MUFU)
template <int HD, bool CAUSAL, bool MAT, int PE = 0>
__global__ void __launch_bounds__(384, 1)
    fa_fwd_pp(const __grid_constant__ CUtensorMap map_qkv, AttnArgs a) {
  using Cfg = PpCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* Qs = smem;
  uint8_t* KVs = smem + Cfg::KV_OFF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;
  uint64_t* kv_empty = bar + 5;
  uint64_t* s_full = bar + 9;
  uint64_t* p_full = bar + 11;
  uint64_t* o_full = bar + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 15);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * 256;
  const int hl = blockIdx.y / (int)a.b, bj = blockIdx.y % (int)a.b;
  const int S = (int)a.s;
  const bool two = q0 + 128 < S;
  const int nkv0 = (CAUSAL && !MAT) ? min(S, q0 + 128) / 128 : S / 128;
  const int nkv1 = two ? ((CAUSAL && !MAT) ? min(S, q0 + 256) / 128 : S / 128) : 0;
  const int nkv = max(nkv0, nkv1);
  constexpr int PASSES = MAT ? 2 : 1;  // MAT: nkv0 == nkv1 (or tile 1 empty)
  const int qcol = (int)(a.qoff + (int64_t)hl * HD), kcol = (int)(a.koff + (int64_t)hl * HD),
            vcol = (int)(a.voff + (int64_t)hl * HD);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < Cfg::KVS; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 4);
      mbar_init(&o_full[t], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc_warp(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp < 4) {
    regs_dec<56>();
    if (warp == 0 && lane == 0) {
      // ---------------------------------------------- TMA producer
      mbar_expect_tx(q_full, (two ? 2 : 1) * Cfg::TILE);
      for (int at = 0; at < Cfg::ATOMS; ++at)
        tma_load_3d(Qs + at * kAtomBytes, &map_qkv, q_full, qcol + 64 * at, bj, q0);
      if (two)
        for (int at = 0; at < Cfg::ATOMS; ++at)
          tma_load_3d(Qs + Cfg::TILE + at * kAtomBytes, &map_qkv, q_full, qcol + 64 * at, bj, q0 + 128);
      for (int u = 0; u < PASSES * nkv; ++u) {  // step u: key tile u % nkv of pass u / nkv
        const int st = u % Cfg::KVS, j = u % nkv;
        const bool with_v = u >= (PASSES - 1) * nkv;  // V only in the last pass
        mbar_wait(&kv_empty[st], ((u / Cfg::KVS) & 1) ^ 1);
        uint8_t* Kt = KVs + st * 2 * Cfg::TILE;
        uint8_t* Vt = Kt + Cfg::TILE;
        mbar_expect_tx(&kv_full[st], (with_v ? 2 : 1) * Cfg::TILE);
        for (int at = 0; at < Cfg::ATOMS; ++at)
          tma_load_3d(Kt + at * kAtomBytes, &map_qkv, &kv_full[st], kcol + 64 * at, bj, j * 128);
        if (with_v)
          for (int at = 0; at < Cfg::ATOMS; ++at)
            tma_load_3d(Vt + at * kAtomBytes, &map_qkv, &kv_full[st], vcol + 64 * at, bj, j * 128);
      }
    } else if (warp == 1) {
      // ---------------------------------------------- MMA issuer (whole warp, elected lane)
      constexpr uint32_t idesc_s = make_idesc(128, 128, false, false);
      constexpr uint32_t idesc_o = make_idesc(128, HD, false, true);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int t, int j) {  // S_t = Q_t · K(j)ᵀ
        const int st = j % Cfg::KVS;
        mbar_wait(&kv_full[st], (j / Cfg::KVS) & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(Qs + t * Cfg::TILE);
        const uint32_t kb = smem_u32(KVs + st * 2 * Cfg::TILE);
        // descriptors built once per tile; each K step only advances the 14-bit start-address
        // field (addresses < 256 KB: no carry out of it), one add instead of the shift / mask
        // chain per descriptor
        const uint64_t qd = smem_desc(qa, 16, 1024), kd = smem_desc(kb, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * kAtomBytes + (kk & 3) * 32) >> 4;
          umma_bf16_w(tmem + t * 128, desc_add(qd, off), desc_add(kd, off), idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit_w(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P̃_t (TMEM, over S_t's first 64 columns) · V(j)
        const int st = j % Cfg::KVS;
        const int jp = MAT ? j - nkv : j;  // key tile within the PV pass
        mbar_wait(&p_full[t], j & 1);
        tc_fence_after();
        const uint32_t vb = smem_u32(KVs + st * 2 * Cfg::TILE + Cfg::TILE);
        const uint64_t vd = smem_desc(vb, kAtomBytes, 1024);
#pragma unroll
        for (int kk = 0; kk < 128 / 16; ++kk)
          umma_bf16_ts_w(tmem + Cfg::O_COL + t * HD, tmem + t * 128 + kk * 8,
                         desc_add(vd, kk * (2048 >> 4)), idesc_o, (jp | kk) != 0 ? 1u : 0u);
      };
      // step u of tile t (u < PASSES·n_t): S_t(u) from stage u; in the last pass P̃_t(u)·V,
      // in MAT's first pass only the wait for the softmax to have read S_t(u)
      if (nkv0 > 0) issue_s(0, 0);
      if (nkv1 > 0) issue_s(1, 0);
      if constexpr (MAT) {
        for (int u = 0; u < 2 * nkv; ++u) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int n = 2 * (t == 0 ? nkv0 : nkv1);
            if (u < n) {
              if (u >= n / 2) issue_pv(t, u);
              else mbar_wait(&p_full[t], u & 1);
              if (u + 1 < n) issue_s(t, u + 1);
              else umma_commit_w(&o_full[t]);
            }
          }
          umma_commit_w(&kv_empty[u % Cfg::KVS]);  // both tiles' products of stage u issued
        }
      } else {
        for (int j = 0; j < nkv; ++j) {
          if (j < nkv0) {
            issue_pv(0, j);
            if (j + 1 < nkv0) issue_s(0, j + 1);
            else umma_commit_w(&o_full[0]);
          }
          if (j < nkv1) {
            issue_pv(1, j);
            if (j + 1 < nkv1) issue_s(1, j + 1);
            else umma_commit_w(&o_full[1]);
          }
          umma_commit_w(&kv_empty[j % Cfg::KVS]);  // both tiles' products of stage j issued
        }
      }
    }
  } else {
    regs_inc<224>();
    // ---------------------------------------------- softmax: one thread per query row
    const int t = (warp - 4) >> 2;
    const int qd = warp & 3;
    const int row = qd * 32 + lane;
    const int q0t = q0 + 128 * t;
    const int qr = q0t + row;
    const int nk = t == 0 ? nkv0 : nkv1;
    const uint32_t tl = tmem + ((uint32_t)(qd * 32) << 16);
    const uint32_t scol = (uint32_t)(t * 128), ocol = (uint32_t)(Cfg::O_COL + t * HD);
    const float sl2 = a.scale * kLog2e;
    const bool drop_on = a.drop.thresh != 0;
    const int W = S / 32;
    const int64_t brow = ((int64_t)hl * a.b + bj) * a.s;
    const uint4* kw = reinterpret_cast<const uint4*>(a.keepbits + (brow + (qr < S ? qr : 0)) * W);
    float m_used = -INFINITY;
    uint64_t l2 = f32x2(0.f, 0.f);
    uint4 wnext = make_uint4(~0u, ~0u, ~0u, ~0u);
    if (drop_on && nk > 0) wnext = kw[0];
    auto load_s = [&](uint32_t (&r)[128]) {
      tmem_ld32_nw(tl + scol, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tmem_ld32_nw(tl + scol + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
      tmem_ld32_nw(tl + scol + 64, *reinterpret_cast<uint32_t(*)[32]>(&r[64]));
      tmem_ld32_nw(tl + scol + 96, *reinterpret_cast<uint32_t(*)[32]>(&r[96]));
      tmem_wait();
    };
    auto row_max = [&](const uint32_t (&r)[128]) {
      float c0 = max3f(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]));
      float c1 = max3f(__uint_as_float(r[3]), __uint_as_float(r[4]), __uint_as_float(r[5]));
#pragma unroll
      for (int i = 6; i < 126; i += 4) {
        c0 = max3f(c0, __uint_as_float(r[i]), __uint_as_float(r[i + 1]));
        c1 = max3f(c1, __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
      }
      return max3f(c0, c1, fmaxf(__uint_as_float(r[126]), __uint_as_float(r[127])));
    };
    if constexpr (MAT) {
      // ---- pass 1: exact row max and sum (no O to rescale: the reference point always moves)
      for (int j = 0; j < nk; ++j) {
        mbar_wait(&s_full[t], j & 1);
        tc_fence_after();
        uint32_t r[128];
        load_s(r);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);  // S_t read: the next Q·Kᵀ may overwrite it
        if (CAUSAL && j * 128 + 127 > q0t) {
          const int k0 = j * 128;
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (k0 + i > qr) r[i] = __float_as_uint(-INFINITY);
        }
        const float mt = row_max(r) * sl2;
        if (mt > m_used) {
          if (m_used != -INFINITY) {
            const float f = ex2f(m_used - mt);
            l2 = fmul2(l2, f32x2(f, f));
          }
          m_used = mt;
        }
        if (m_used == -INFINITY) continue;  // every key so far masked
        const uint64_t sl2x2 = f32x2(sl2, sl2), nmm2 = f32x2(-m_used, -m_used);
#pragma unroll
        for (int i = 0; i < 128; i += 2) {
          float x0, x1;
          f32x2_split(ffma2(f32x2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2, nmm2), x0, x1);
          l2 = fadd2(l2, f32x2(ex2f(x0), ex2f(x1)));
        }
      }
      // ---- pass 2: normalised P, mask, P̃ -> the stored interior; P̃ -> TMEM for O += P̃·V
      float le, lo;
      f32x2_split(l2, le, lo);
      const float inv_l = 1.f / (le + lo), ik = a.drop.inv_keep;
      const float mm = m_used == -INFINITY ? 0.f : m_used;
      const uint64_t sl2x2 = f32x2(sl2, sl2), nmm2 = f32x2(-mm, -mm);
      const int64_t irow = (brow + qr) * (int64_t)S;
      for (int j = 0; j < nk; ++j) {
        const uint4 wcur = wnext;
        if (drop_on && j + 1 < nk) wnext = kw[j + 1];
        const int u = nk + j;
        mbar_wait(&s_full[t], u & 1);
        tc_fence_after();
        uint32_t r[128];
        load_s(r);
        const uint32_t words[4] = {wcur.x, wcur.y, wcur.z, wcur.w};
        const int k0 = j * 128;
        const bool diag = CAUSAL && k0 + 127 > q0t;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t pk[32], pm[32];
#pragma unroll
          for (int i = 64 * hh; i < 64 * hh + 64; i += 2) {
            float x0, x1;
            f32x2_split(ffma2(f32x2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2, nmm2), x0, x1);
            float p0 = ex2f(x0) * inv_l, p1 = ex2f(x1) * inv_l;
            if (CAUSAL) {
              if (diag && k0 + i > qr) p0 = 0.f;
              if (diag && k0 + i + 1 > qr) p1 = 0.f;
            }
            const uint32_t w = words[i >> 5];
            const float d0 = (w >> (i & 31)) & 1u ? p0 * ik : 0.f;
            const float d1 = (w >> ((i + 1) & 31)) & 1u ? p1 * ik : 0.f;
            pm[(i - 64 * hh) >> 1] = pack_bf16x2(p0, p1);
            pk[(i - 64 * hh) >> 1] = pack_bf16x2(d0, d1);
          }
          uint8_t* smo = reinterpret_cast<uint8_t*>(static_cast<bf16*>(a.sm) + irow + k0 + 64 * hh);
          uint8_t* sdo = reinterpret_cast<uint8_t*>(static_cast<bf16*>(a.sd) + irow + k0 + 64 * hh);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            st_v8(smo + 32 * v, pm[8 * v], pm[8 * v + 1], pm[8 * v + 2], pm[8 * v + 3], pm[8 * v + 4],
                  pm[8 * v + 5], pm[8 * v + 6], pm[8 * v + 7]);
            st_v8(sdo + 32 * v, pk[8 * v], pk[8 * v + 1], pk[8 * v + 2], pk[8 * v + 3], pk[8 * v + 4],
                  pk[8 * v + 5], pk[8 * v + 6], pk[8 * v + 7]);
          }
#pragma unroll
          for (int v = 0; v < 2; ++v) {  // 32 keys -> 32 mask bytes (the raw keep bit)
            const uint32_t wb = words[2 * hh + v];
            uint32_t q8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const uint32_t bits = (wb >> (4 * e)) & 0xFu;
              q8[e] = (bits & 1u) | ((bits & 2u) << 7) | ((bits & 4u) << 14) | ((bits & 8u) << 21);
            }
            st_v8(a.mask + irow + k0 + 64 * hh + 32 * v, q8[0], q8[1], q8[2], q8[3], q8[4], q8[5],
                  q8[6], q8[7]);
          }
          tmem_st32u(tl + scol + 32 * hh, pk);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
      }
    }
    for (int j = 0; j < (MAT ? 0 : nk); ++j) {
      const uint4 wcur = wnext;
      if (drop_on && j + 1 < nk) wnext = kw[j + 1];  // next tile's keep words, one tile ahead
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      uint32_t r[128];
      tmem_ld32_nw(tl + scol, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tmem_ld32_nw(tl + scol + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
      tmem_ld32_nw(tl + scol + 64, *reinterpret_cast<uint32_t(*)[32]>(&r[64]));
      tmem_ld32_nw(tl + scol + 96, *reinterpret_cast<uint32_t(*)[32]>(&r[96]));
      tmem_wait();
      if (CAUSAL && j * 128 + 127 > q0t) {  // the diagonal tile: keys past the query masked
        const int k0 = j * 128;
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (k0 + i > qr) r[i] = __float_as_uint(-INFINITY);
      }
      // row max of the raw scores (the scale is positive: max(s)·c == max(s·c) exactly)
      float cm;
      {
        float c0 = max3f(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]));
        float c1 = max3f(__uint_as_float(r[3]), __uint_as_float(r[4]), __uint_as_float(r[5]));
#pragma unroll
        for (int i = 6; i < 126; i += 4) {
          c0 = max3f(c0, __uint_as_float(r[i]), __uint_as_float(r[i + 1]));
          c1 = max3f(c1, __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
        }
        cm = max3f(c0, c1, fmaxf(__uint_as_float(r[126]), __uint_as_float(r[127])));
      }
      const float mt = cm * sl2;
      float f = 1.f;
      bool rescale = false;
      if (m_used == -INFINITY) {
        m_used = mt;
      } else if (mt > m_used + 8.f) {
        f = ex2f(m_used - mt);
        m_used = mt;
        l2 = fmul2(l2, f32x2(f, f));
        rescale = true;
      }
      if (__any_sync(0xffffffffu, rescale)) {
        // P̃_t(j-1)·V completed before S_t(j) was signalled (issued earlier, same commit chain)
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          float o[32];
          tmem_ld32(tl + ocol + c * 32, o);
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= f;
          tmem_st32(tl + ocol + c * 32, o);
        }
      }
      const float mm = m_used == -INFINITY ? 0.f : m_used;
      const uint64_t sl2x2 = f32x2(sl2, sl2), nmm2 = f32x2(-mm, -mm);
      const uint32_t words[4] = {wcur.x, wcur.y, wcur.z, wcur.w};
      uint32_t pk[64];
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        float x0, x1;
        const uint64_t x2 = ffma2(f32x2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sl2x2, nmm2);
        float p0, p1;
        if constexpr (PE > 0) {
          if ((i >> 1) % PE == PE - 1) {
            const uint64_t e2 = ex2_poly2(x2);
            l2 = fadd2(l2, e2);
            f32x2_split(e2, p0, p1);
          } else {
            f32x2_split(x2, x0, x1);
            p0 = ex2f(x0), p1 = ex2f(x1);
            l2 = fadd2(l2, f32x2(p0, p1));
          }
        } else {
          f32x2_split(x2, x0, x1);
          p0 = ex2f(x0), p1 = ex2f(x1);
          l2 = fadd2(l2, f32x2(p0, p1));
        }
        const uint32_t w = words[i >> 5];
        pk[i >> 1] = pack_bf16x2((w >> (i & 31)) & 1u ? p0 : 0.f, (w >> ((i + 1) & 31)) & 1u ? p1 : 0.f);
      }
      tmem_st32u(tl + scol, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
      tmem_st32u(tl + scol + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    if (nk > 0) {  // epilogue: O · (1/(1-p))/l -> bf16; LSE
      float le, lo;
      f32x2_split(l2, le, lo);
      const float l = le + lo;
      const float oscale = MAT ? 1.f : a.drop.inv_keep / l;  // MAT: P̃ was normalised
      mbar_wait(&o_full[t], 0);
      tc_fence_after();
      // O rows are HD·2 bytes apart from the next query's by b·ldo elements: one thread per row
      // would issue 32 scattered 16-byte stores per instruction. Stage the warp's 32 rows in
      // Q_t's shared memory (free: its last Q·Kᵀ completed before o_full) — 128 / 256-byte rows,
      // 16-byte chunks XOR-swizzled by row — then store them row-contiguously.
      constexpr int CH = HD / 8;  // 16-byte chunks per row
      uint8_t* stage = Qs + t * Cfg::TILE + qd * 32 * Cfg::ORS;
      uint8_t* srow = stage + lane * Cfg::ORS;
#pragma unroll 1
      for (int c = 0; c < HD / 32; ++c) {
        float v[32];
        tmem_ld32(tl + ocol + c * 32, v);
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          const int ch = (c * 32 + i) / 8;
          *reinterpret_cast<uint4*>(srow + ((ch ^ (lane & 7)) * 16)) =
              make_uint4(pack_bf16x2(v[i] * oscale, v[i + 1] * oscale), pack_bf16x2(v[i + 2] * oscale, v[i + 3] * oscale),
                         pack_bf16x2(v[i + 4] * oscale, v[i + 5] * oscale), pack_bf16x2(v[i + 6] * oscale, v[i + 7] * oscale));
        }
      }
      __syncwarp();
      bf16* obase = static_cast<bf16*>(a.o) + (int64_t)bj * a.ldo + (int64_t)hl * HD;
#pragma unroll 1
      for (int idx = lane; idx < 32 * CH; idx += 32) {
        const int r = idx / CH, ch = idx % CH;
        const int q = q0t + qd * 32 + r;
        if (q < S)
          *reinterpret_cast<uint4*>(obase + (int64_t)q * a.b * a.ldo + ch * 8) =
              *reinterpret_cast<const uint4*>(stage + r * Cfg::ORS + ((ch ^ (r & 7)) * 16));
      }
      if (qr < S && a.lse) a.lse[brow + qr] = (m_used + log2f(l)) * kLn2;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, 512);
  }
}

template <int HD, bool CAUSAL, bool MAT, int PE>
void launch_pp_pe(const AttnArgs& a, cudaStream_t st) {
  using Cfg = PpCfg<HD>;
  static bool once = [] {
    SPL_CUDA(cudaFuncSetAttribute(fa_fwd_pp<HD, CAUSAL, MAT, PE>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    return true;
  }();
  (void)once;
  const CUtensorMap mq = attn_seq_map(a.qkv, a.ld, a.b, a.s, a.ld, 128);
  dim3 grid((unsigned)((a.s + 255) / 256), (unsigned)(a.lh * a.b));
  fa_fwd_pp<HD, CAUSAL, MAT, PE><<<grid, 384, Cfg::SMEM, st>>>(mq, a);
  SPL_CHECK_LAUNCH();
}

// SPL_ATTN_POLY=n (0, 2, 4, 8): every n-th exponential pair of the recompute regimes' forward
// on the FMA pipe (A/B switch; the default is the measured one)
int poly_period() {
  static const int pe = [] {
    const char* e = std::getenv("SPL_ATTN_POLY");
    const int v = e ? std::atoi(e) : kPolyDefault;
    return (v == 2 || v == 4 || v == 8) ? v : 0;
  }();
  return pe;
}

template <int HD, bool CAUSAL, bool MAT>
void launch_pp(const AttnArgs& a, cudaStream_t st) {
  if constexpr (!MAT) {
    switch (poly_period()) {
      case 2: return launch_pp_pe<HD, CAUSAL, MAT, 2>(a, st);
      case 4: return launch_pp_pe<HD, CAUSAL, MAT, 4>(a, st);
      case 8: return launch_pp_pe<HD, CAUSAL, MAT, 8>(a, st);
      default: break;
    }
  }
  launch_pp_pe<HD, CAUSAL, MAT, 0>(a, st);
}

}  // namespace

bool attn_fwd_pp_supported(const AttnArgs& a) {
  static const bool off = [] {
    const char* e = std::getenv("SPL_ATTN_FWD_PP");
    return e != nullptr && e[0] == '0';
  }();
  const bool regime_ok = a.sm == nullptr
                             ? a.lse != nullptr
                             : (a.mask != nullptr && a.sd != nullptr && ((uintptr_t)a.sm & 31) == 0 &&
                                ((uintptr_t)a.sd & 31) == 0 && ((uintptr_t)a.mask & 31) == 0);
  return !off && regime_ok && a.keep_t == 0 &&
         (a.hd == 64 || a.hd == 96 || a.hd == 128) && a.s % 128 == 0 && a.s < (1 << 30) &&
         a.ld % 8 == 0 && a.ldo % 8 == 0 && ((uintptr_t)a.qkv & 15) == 0 &&
         ((uintptr_t)a.o & 15) == 0 && (a.keepbits != nullptr || a.drop.thresh == 0) &&
         (a.keepbits == nullptr || ((uintptr_t)a.keepbits & 15) == 0);
}

void attn_fwd_pp(const AttnArgs& a, cudaStream_t st) {
  switch (a.hd) {
#define SPL_PP_CASE(HDX)                                                                    \
  case HDX:                                                                                 \
    if (a.sm != nullptr)                                                                    \
      return a.causal ? launch_pp<HDX, true, true>(a, st) : launch_pp<HDX, false, true>(a, st); \
    return a.causal ? launch_pp<HDX, true, false>(a, st) : launch_pp<HDX, false, false>(a, st);
    SPL_PP_CASE(64)
    SPL_PP_CASE(96)
    SPL_PP_CASE(128)
#undef SPL_PP_CASE
    default: raise(3, "attn_fwd_pp: unsupported head_dim");
  }
}

}  // namespace spl::k
