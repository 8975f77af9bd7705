// bf16 GEMM on the 5th-generation tensor cores (sm_100a): TMA -> shared memory (128B swizzle)
// -> tcgen05.mma (single elected thread) -> fp32 accumulator in TMEM -> tcgen05.ld epilogue
// with the fused layer epilogues (bias, bias+GELU dual output, GELU-backward, fp32 wgrad).
//
// One kernel template covers the three GEMM orientations of the layer
// (C[M,N] = A[M,K]·B[K,N]):
//   forward  (QKV, proj, FC1, FC2):  A K-major (activations),  B MN-major (weights [in,out])
//   dgrad    (dY·Wᵀ):                A K-major,                 B K-major
//   wgrad    (Xᵀ·dY):                A MN-major,                B MN-major
// The majorness is a UMMA instruction-descriptor bit plus the matching smem descriptor
// (LBO/SBO) and TMA box, so no operand is ever transposed in memory.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
// warps 2..5 = epilogue (warp w reads TMEM lanes 32*(w%4)..+31 = tile rows).
// Tile 128 x BN x 64, STAGES-deep mbarrier ring between TMA and MMA.
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "gemm_epilogue.cuh"
#include "tc_common.cuh"

namespace spl::k {

namespace {

using namespace tc;

constexpr int BM = 128, BK = 64, UK = 16;
constexpr int kThreads = 192;

template <int BN>
struct TileCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = BN;  // fp32 accumulator, one column per N
};

// ------------------------------------------------------------------ fast GELU for the bf16 epilogues
// erf from Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7, far below the bf16 rounding of the
// outputs): one ex2 and one reciprocal on the MUFU pipe plus six FMAs, and the GELU derivative
// shares the exponential with the normal pdf. erff's longer FMA chain in the epilogue cost the
// GELU'-fused FC2 dgrad ~14 % of its throughput under the power cap (tools/gemm_bench.py).
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// returns erf(x / sqrt 2); *e_out = exp(-x^2 / 2)
__device__ __forceinline__ float erf_scaled(float x, float* e_out) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float e = __expf(-z * z);
  const float t = rcp_approx(fmaf(0.3275911f, z, 1.f));
  const float poly =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f),
               0.254829592f);
  *e_out = e;
  return copysignf(1.f - poly * e, x);
}
__device__ __forceinline__ float gelu_fast(float x) {
  float e;
  return 0.5f * x * (1.f + erf_scaled(x, &e));
}
__device__ __forceinline__ float gelu_grad_fast(float x) {
  float e;
  const float cdf = 0.5f * (1.f + erf_scaled(x, &e));
  return fmaf(x * 0.3989422804014327f, e, cdf);
}

// ------------------------------------------------------------------ epilogue store
// 32-byte global store (st.global.v8.b32, sm_100): one full sector per lane. p 32-byte aligned.
__device__ __forceinline__ void st_v8a(void* p, const uint32_t (&w)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
__device__ __forceinline__ uint32_t pk_bf16(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&t);
}
template <int EPI>
__device__ __forceinline__ void store_chunk(const GemmArgs& g, int64_t m, int64_t n0,
                                            const float (&v)[32]) {
  if (m >= g.M) return;
  const bool full = n0 + 32 <= g.N;
  if constexpr (EPI == (int)Epi::F32) {
    float* c = gemm_row<float>(g, m) + n0;
    if (full) {
      if (g.accumulate) {  // running fp32 sum over microbatches: C_old + (this GEMM)
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 o = *reinterpret_cast<const float4*>(c + i);
          *reinterpret_cast<float4*>(c + i) =
              make_float4(o.x + v[i], o.y + v[i + 1], o.z + v[i + 2], o.w + v[i + 3]);
        }
      } else if (((uintptr_t)c & 31) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint32_t w[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) w[j] = __float_as_uint(v[i + j]);
          st_v8a(c + i, w);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
    } else {
      for (int i = 0; i < 32 && n0 + i < g.N; ++i) c[i] = g.accumulate ? c[i] + v[i] : v[i];
    }
    return;
  } else {
    float o[32];
    float o2[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = v[i];
    if constexpr (EPI == (int)Epi::Bias || EPI == (int)Epi::BiasGelu) {
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 b = *reinterpret_cast<const float4*>(g.bias + n0 + i);
          o[i] += b.x; o[i + 1] += b.y; o[i + 2] += b.z; o[i + 3] += b.w;
        }
      } else {
        for (int i = 0; i < 32 && n0 + i < g.N; ++i) o[i] += g.bias[n0 + i];
      }
    }
    if constexpr (EPI == (int)Epi::BiasGelu) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float pre = __bfloat162float(__float2bfloat16_rn(o[i]));
        o2[i] = gelu_fast(pre);
      }
    }
    if constexpr (EPI == (int)Epi::GeluBwd) {
      const bf16* ax = static_cast<const bf16*>(g.aux) + m * g.ldaux + n0;
      if (full) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          const uint4 t = *reinterpret_cast<const uint4*>(ax + i);
          const bf16* e = reinterpret_cast<const bf16*>(&t);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[i + j] *= gelu_grad_fast(__bfloat162float(e[j]));
        }
      } else {
        for (int i = 0; i < 32 && n0 + i < g.N; ++i) o[i] *= gelu_grad_fast(__bfloat162float(ax[i]));
      }
    }
    bf16* c = gemm_row<bf16>(g, m) + n0;
    bf16* c2 = EPI == (int)Epi::BiasGelu ? static_cast<bf16*>(g.C2) + m * g.ldc + n0 : nullptr;
    if (full && (((uintptr_t)c | (uintptr_t)(c2 != nullptr ? c2 : c)) & 31) == 0) {
      // a row's 32 columns as two 32-byte stores per output (full sectors)
#pragma unroll
      for (int i = 0; i < 32; i += 16) {
        uint32_t w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w[j] = pk_bf16(o[i + 2 * j], o[i + 2 * j + 1]);
        st_v8a(c + i, w);
        if constexpr (EPI == (int)Epi::BiasGelu) {
#pragma unroll
          for (int j = 0; j < 8; ++j) w[j] = pk_bf16(o2[i + 2 * j], o2[i + 2 * j + 1]);
          st_v8a(c2 + i, w);
        }
      }
    } else if (full) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 t;
        bf16* e = reinterpret_cast<bf16*>(&t);
#pragma unroll
        for (int j = 0; j < 8; ++j) e[j] = __float2bfloat16_rn(o[i + j]);
        *reinterpret_cast<uint4*>(c + i) = t;
        if constexpr (EPI == (int)Epi::BiasGelu) {
#pragma unroll
          for (int j = 0; j < 8; ++j) e[j] = __float2bfloat16_rn(o2[i + j]);
          *reinterpret_cast<uint4*>(c2 + i) = t;
        }
      }
    } else {
      for (int i = 0; i < 32 && n0 + i < g.N; ++i) {
        c[i] = __float2bfloat16_rn(o[i]);
        if constexpr (EPI == (int)Epi::BiasGelu) c2[i] = __float2bfloat16_rn(o2[i]);
      }
    }
  }
}

// ------------------------------------------------------------------ the kernel
// Grouped tile order: `group` consecutive M blocks sweep all N blocks, so the A row-panels of
// a group stay in L2 while the B tiles stream through. The host sizes the group so the panels
// take ~48 MB of the 126 MB L2: B is then re-read tiles_m/group times instead of tiles_m/8
// (measured 3.5 GB -> see profiles/ for the per-launch DRAM bytes).
__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int group, int& mb,
                                            int& nb) {
  const int per_group = group * tiles_n;
  const int g = tile / per_group;
  const int first_m = g * group;
  const int gsize = min(tiles_m - first_m, group);
  const int r = tile % per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

// Persistent: one CTA per SM loops over output tiles. Two TMEM accumulators (2 x BN fp32
// columns) let the epilogue of tile i overlap the MMA main loop of tile i+1.
template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, const GemmArgs g, int tiles_m,
                   int tiles_n, int group) {
  using Cfg = TileCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* tiles = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + Cfg::STAGES;
  uint64_t* tfull = empty_bar + Cfg::STAGES;  // [2]
  uint64_t* tempty = tfull + 2;               // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (int)((g.K + BK - 1) / BK);
  const int ntiles = tiles_m * tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"((uint32_t)(2 * Cfg::TMEM_COLS)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(tile, tiles_m, tiles_n, group, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (uint32_t)(it / Cfg::STAGES) & 1u;
          mbar_wait(&empty_bar[s], ph ^ 1u);
          uint8_t* sa = tiles + s * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_expect_tx(&full_bar[s], Cfg::STAGE_BYTES);
          const int k0 = kb * BK;
          if (A_MN) {  // [K rows][M cols]: two 64-wide M atoms of 64 k-rows
            tma_load_2d(sa, &map_a, &full_bar[s], m0, k0);
            tma_load_2d(sa + 8192, &map_a, &full_bar[s], m0 + 64, k0);
          } else {  // [M rows][K cols]: one 128-row box
            tma_load_2d(sa, &map_a, &full_bar[s], k0, m0);
          }
          if (B_MN) {  // [K rows][N cols]: BN/64 atoms
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sb + j * 8192, &map_b, &full_bar[s], n0 + 64 * j, k0);
          } else {  // [N rows][K cols]: one BN-row box
            tma_load_2d(sb, &map_b, &full_bar[s], k0, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = make_idesc(BM, BN, A_MN, B_MN);
      int it = 0, local = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t aph = (uint32_t)(local >> 1) & 1u;
        mbar_wait(&tempty[acc], aph ^ 1u);  // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t tacc = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t ph = (uint32_t)(it / Cfg::STAGES) & 1u;
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(tiles + s * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            // K-major: advance 16 elements (32 B) inside the 128 B swizzle row;
            // MN-major: advance 16 k-rows (2 KB), i.e. two 8-row core-matrix groups.
            const uint64_t ad = A_MN ? smem_desc(sa + kk * 2048, 8192, 1024)
                                     : smem_desc(sa + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc(sb + kk * 2048, 8192, 1024)
                                     : smem_desc(sb + kk * 32, 16, 1024);
            umma_bf16(tacc, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          umma_commit(&empty_bar[s]);  // frees the smem stage once these MMAs have read it
        }
        umma_commit(&tfull[acc]);  // accumulator complete
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> fused op -> global
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = q * 32 + lane;
    int local = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++local) {
      int mb, nb;
      tile_coords(tile, tiles_m, tiles_n, group, mb, nb);
      const int64_t m0 = (int64_t)mb * BM, n0 = (int64_t)nb * BN;
      const int acc = local & 1;
      const uint32_t aph = (uint32_t)(local >> 1) & 1u;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
        if (n0 + c * 32 < g.N) store_chunk<EPI>(g, m0 + row, n0 + c * 32, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)(2 * Cfg::TMEM_COLS)));
  }
}

// ------------------------------------------------------------------ CTA-pair variant
// Two CTAs of a cluster (one TPC) compute a 256 x 256 tile with tcgen05.mma.cta_group::2:
// CTA r stages A rows m0+128r..+127 and B columns n0+128r..+127; the leader (rank 0) issues
// the M=256 MMAs, which read both CTAs' shared memory, and each CTA's TMEM receives its own
// 128 rows x 256 columns. Per SM the shared-memory operand traffic per MMA drops from
// A 16 KB + B 32 KB to 16 KB + 16 KB per 64-deep k block.
// Barriers: full[s] lives in the leader and counts both CTAs' TMA bytes; empty[s] and
// tfull[acc] exist in both CTAs and are arrived by the leader's multicast commits; tempty[acc]
// lives in the leader and collects the 4+4 epilogue warps of the pair.
// TN (pair tile width) 256, or 128 for GEMMs whose 256-wide tiles fill the 74 CTA pairs' last
// wave badly (t > 1 shards: N = 3h/t, 4h/t, h/t); each CTA stages TN/2 columns of B.
constexpr int P_STAGES = 6;
constexpr int P_A_BYTES = 128 * BK * 2;
template <int TN>
constexpr int p_stage_bytes() { return P_A_BYTES + (TN / 2) * BK * 2; }
template <int TN>
constexpr int p_smem() { return P_STAGES * p_stage_bytes<TN>() + 1024 + 256; }

// Tensor maps of the pair kernel: one per operand, or one per row block of a sharded operand.
struct PairMaps {
  CUtensorMap a[GemmArgs::kMaxShards];
  CUtensorMap b[GemmArgs::kMaxShards];
};
// Map and token coordinate of a (possibly sharded) operand: block q = c / rows.
__device__ __forceinline__ const CUtensorMap* shard_map(const CUtensorMap* maps, int n, int rows,
                                                        int& c) {
  if (n <= 1) return maps;
  const int q = c / rows;
  c -= q * rows;
  return maps + q;
}

template <bool A_MN, bool B_MN, int EPI, int TN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_tc_pair_kernel(const __grid_constant__ PairMaps maps, const GemmArgs g, int tiles_m,
                        int tiles_n, int group, int l2_hint) {
  static_assert(TN == 256 || TN == 128, "pair tile width");
  constexpr int P_STAGE_BYTES = p_stage_bytes<TN>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* tiles = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE_BYTES);
  uint64_t* empty_bar = full_bar + P_STAGES;
  uint64_t* tfull = empty_bar + P_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int nk = (int)((g.K + BK - 1) / BK);
  const int ntiles = tiles_m * tiles_n;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // one arrive per epilogue warp of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < (g.a_shards > 1 ? g.a_shards : 1); ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.a[i]) : "memory");
    for (int i = 0; i < (g.b_shards > 1 ? g.b_shards : 1); ++i)
      asm volatile("prefetch.tensormap [%0];" ::"l"(&maps.b[i]) : "memory");
  }
  // Both CTAs must be running before the 2-CTA TMEM allocation: its handshake writes into the
  // peer's shared memory, and a peer that has not started yet (its SM still busy with another
  // stream's kernel) loses it and waits forever — an intermittent hang seen under concurrency.
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"((uint32_t)(2 * TN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs), bytes counted on the leader's full[s]
      int it = 0, local = 0;
      const uint64_t pol_a = (l2_hint & 1) ? l2_policy_evict_last() : l2_policy_evict_normal();
      const bool ksnake = (l2_hint & 2) != 0;
      for (int tile = pair; tile < ntiles; tile += npairs, ++local) {
        int mb, nb;
        tile_coords(tile, tiles_m, tiles_n, group, mb, nb);
        const int m0 = mb * 256 + 128 * (int)rank, n0 = nb * TN + (TN / 2) * (int)rank;
        // K snake: odd waves walk K backwards, so they start on the k-blocks the previous wave
        // loaded last (still in L2) for the panels the two waves share
        const bool rev = ksnake && (local & 1);
        for (int kbi = 0; kbi < nk; ++kbi, ++it) {
          const int kb = rev ? nk - 1 - kbi : kbi;
          const int s = it % P_STAGES;
          const uint32_t ph = (uint32_t)(it / P_STAGES) & 1u;
          mbar_wait(&empty_bar[s], ph ^ 1u);
          uint8_t* sa = tiles + s * P_STAGE_BYTES;
          uint8_t* sb = sa + P_A_BYTES;
          if (rank == 0) mbar_expect_tx(&full_bar[s], 2 * P_STAGE_BYTES);
          const uint32_t fb = mapa_rank(smem_u32(&full_bar[s]), 0);
          const int k0 = kb * BK;
          // A panels are reused across the whole N sweep of a raster group: evict_last keeps
          // them in L2 while B tiles and the epilogue's output stream through
          // sharded operands: the token coordinate (A: K when MN-major, else M; B: K when
          // MN-major) selects the row block, i.e. the rank whose shard holds these rows
          const int sr = (int)g.shard_rows;
          if (A_MN) {
            int ka = k0;
            const CUtensorMap* ma = shard_map(maps.a, g.a_shards, sr, ka);
            tma_load_2d_pair_hint(sa, ma, fb, m0, ka, pol_a);
            tma_load_2d_pair_hint(sa + 8192, ma, fb, m0 + 64, ka, pol_a);
          } else {
            int ma0 = m0;
            const CUtensorMap* ma = shard_map(maps.a, g.a_shards, sr, ma0);
            tma_load_2d_pair_hint(sa, ma, fb, k0, ma0, pol_a);
          }
          if (B_MN) {
            int kb0 = k0;
            const CUtensorMap* mbp = shard_map(maps.b, g.b_shards, sr, kb0);
            tma_load_2d_pair(sb, mbp, fb, n0, kb0);
            if (TN == 256) tma_load_2d_pair(sb + 8192, mbp, fb, n0 + 64, kb0);
          } else {
            tma_load_2d_pair(sb, &maps.b[0], fb, k0, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader only)
      constexpr uint32_t idesc = make_idesc(256, TN, A_MN, B_MN);
      int it = 0, local = 0;
      for (int tile = pair; tile < ntiles; tile += npairs, ++local) {
        const int acc = local & 1;
        const uint32_t aph = (uint32_t)(local >> 1) & 1u;
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t tacc = tmem_base + (uint32_t)(acc * TN);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % P_STAGES;
          const uint32_t ph = (uint32_t)(it / P_STAGES) & 1u;
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(tiles + s * P_STAGE_BYTES);
          const uint32_t sb = sa + P_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = A_MN ? smem_desc(sa + kk * 2048, 8192, 1024)
                                     : smem_desc(sa + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc(sb + kk * 2048, 8192, 1024)
                                     : smem_desc(sb + kk * 32, 16, 1024);
            umma_bf16_pair(tacc, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          umma_commit_pair(&empty_bar[s]);
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else {
    // ---------------- epilogue (both CTAs): this CTA's 128 rows x 256 columns
    const int q = warp & 3;
    const int row = 128 * (int)rank + q * 32 + lane;
    const uint32_t tempty_leader0 = mapa_rank(smem_u32(&tempty[0]), 0);
    int local = 0;
    for (int tile = pair; tile < ntiles; tile += npairs, ++local) {
      int mb, nb;
      tile_coords(tile, tiles_m, tiles_n, group, mb, nb);
      const int64_t m0 = (int64_t)mb * 256, n0 = (int64_t)nb * TN;
      const int acc = local & 1;
      const uint32_t aph = (uint32_t)(local >> 1) & 1u;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < TN / 32; ++c) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * TN + c * 32), v);
        if (n0 + c * 32 < g.N) store_chunk<EPI>(g, m0 + row, n0 + c * 32, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + (uint32_t)(acc * sizeof(uint64_t)));
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)(2 * TN)));
  }
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    SPL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (p == nullptr || q != cudaDriverEntryPointSuccess)
      raise(3, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

struct MapKey {
  const void* ptr;
  uint64_t inner, outer, ld;
  uint32_t box0, box1;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && ld == o.ld && box0 == o.box0 &&
           box1 == o.box1;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    h ^= std::hash<uint64_t>()(k.inner * 1315423911u + k.outer * 2654435761u + k.ld) + 0x9e3779b9 +
         (h << 6) + (h >> 2);
    h ^= (size_t)k.box0 * 31 + k.box1;
    return h;
  }
};

// 2-D bf16 tensor map over a row-major matrix [outer][inner] with row stride ld elements.
CUtensorMap make_map(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box0,
                     uint32_t box1) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  const MapKey key{ptr, inner, outer, ld, box0, box1};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box0, box1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(3, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  return m;
}

// M blocks per raster group, from a DRAM-traffic model of the grouped order: a group's A
// panels (bm x K each) stay in L2 for its whole N sweep if they fit a 48 MB budget, else they
// are re-streamed once per wave (the `workers` concurrent tiles cover workers/group N blocks);
// B panels are re-read once per group. Small K: large groups (A once, B a few times); large K
// (24576 at 22B): groups near sqrt(workers) instead of the 3 that the L2 budget alone allows
// (FC1 dgrad 3.6 -> ~2.3 GB of DRAM traffic per launch).
int pick_group(int64_t K, int bm, int bn, int tiles_m, int tiles_n, int workers) {
  const double pa = (double)bm * K * 2, pb = (double)bn * K * 2;
  const double a_tot = pa * tiles_m, b_tot = pb * tiles_n;
  int best = 1;
  double best_cost = 1e300;
  for (int gm = 1; gm <= tiles_m; ++gm) {
    const int wave_n = std::max(1, workers / gm);
    const double a_reads = gm * pa <= (double)(48ll << 20) ? 1.0 : (double)((tiles_n + wave_n - 1) / wave_n);
    const double b_reads = (double)((tiles_m + gm - 1) / gm);
    const double cost = a_tot * a_reads + b_tot * b_reads;
    if (cost < best_cost * (1 - 1e-9)) {
      best_cost = cost;
      best = gm;
    }
  }
  return best;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
void launch_tc(const GemmArgs& g, cudaStream_t st) {
  using Cfg = TileCfg<BN>;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, EPI>;
  static bool attr = [&] {
    SPL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    return true;
  }();
  (void)attr;
  // A: K-major [M][K] boxes {64, 128}; MN-major [K][M] boxes {64, 64}
  const CUtensorMap ma = A_MN ? make_map(g.A, g.M, g.K, g.lda, 64, BK)
                              : make_map(g.A, g.K, g.M, g.lda, BK, BM);
  const CUtensorMap mb = B_MN ? make_map(g.B, g.N, g.K, g.ldb, 64, BK)
                              : make_map(g.B, g.K, g.N, g.ldb, BK, BN);
  const int tiles_m = (int)((g.M + BM - 1) / BM), tiles_n = (int)((g.N + BN - 1) / BN);
  const int ntiles = tiles_m * tiles_n;
  const int grid = ntiles < kNumSMs ? ntiles : kNumSMs;
  const int group = pick_group(g.K, BM, BN, tiles_m, tiles_n, grid);
  kern<<<grid, kThreads, Cfg::SMEM, st>>>(ma, mb, g, tiles_m, tiles_n, group);
  SPL_CHECK_LAUNCH();
}

template <bool A_MN, bool B_MN, int EPI, int TN>
void launch_pair(const GemmArgs& g, cudaStream_t st) {
  auto kern = gemm_tc_pair_kernel<A_MN, B_MN, EPI, TN>;
  constexpr int P_SMEM = p_smem<TN>();
  static bool attr = [&] {
    SPL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM));
    return true;
  }();
  (void)attr;
  // per-CTA halves: A 128 rows, B 128 columns; a sharded operand gets one map per row block
  PairMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  if (g.a_shards > 1) {
    require(g.a_shards <= GemmArgs::kMaxShards && g.shard_rows % (A_MN ? BK : 128) == 0 &&
                (A_MN ? g.K : g.M) == g.a_shards * g.shard_rows,
            "gemm_tc: sharded A needs row blocks aligned to the tile");
    for (int q = 0; q < g.a_shards; ++q)
      maps.a[q] = A_MN ? make_map(g.a_shard[q], g.M, g.shard_rows, g.lda, 64, BK)
                       : make_map(g.a_shard[q], g.K, g.shard_rows, g.lda, BK, 128);
  } else {
    maps.a[0] = A_MN ? make_map(g.A, g.M, g.K, g.lda, 64, BK)
                     : make_map(g.A, g.K, g.M, g.lda, BK, 128);
  }
  if (g.b_shards > 1) {
    require(B_MN && g.b_shards <= GemmArgs::kMaxShards && g.shard_rows % BK == 0 &&
                g.K == g.b_shards * g.shard_rows,
            "gemm_tc: sharded B must be MN-major with K row blocks aligned to the tile");
    for (int q = 0; q < g.b_shards; ++q)
      maps.b[q] = make_map(g.b_shard[q], g.N, g.shard_rows, g.ldb, 64, BK);
  } else {
    maps.b[0] = B_MN ? make_map(g.B, g.N, g.K, g.ldb, 64, BK)
                     : make_map(g.B, g.K, g.N, g.ldb, BK, TN / 2);
  }
  const int tiles_m = (int)((g.M + 255) / 256), tiles_n = (int)((g.N + TN - 1) / TN);
  const int ntiles = tiles_m * tiles_n;
  const int pairs = ntiles < kNumSMs / 2 ? ntiles : kNumSMs / 2;
  int group = pick_group(g.K, 256, TN, tiles_m, tiles_n, pairs);
  if (const char* e = std::getenv("SPL_GEMM_GROUP")) {  // dev sweeps (tools/gemm_group_sweep.py)
    const int v = std::atoi(e);
    if (v > 0) group = std::min(v, tiles_m);
  }
  static const int l2_hint = [] {
    const char* e = std::getenv("SPL_GEMM_L2HINT");
    const char* k = std::getenv("SPL_GEMM_KSNAKE");
    return ((e != nullptr && e[0] == '0') ? 0 : 1) | ((k != nullptr && k[0] == '0') ? 0 : 2);
  }();
  kern<<<2 * pairs, kThreads, P_SMEM, st>>>(maps, g, tiles_m, tiles_n, group, l2_hint);
  SPL_CHECK_LAUNCH();
}

// BN == 0 / 1 select the CTA-pair kernel with 256 x 256 / 256 x 128 tiles.
template <int BN, bool A_MN, bool B_MN, int EPI>
void run(const GemmArgs& g, cudaStream_t st) {
  if constexpr (BN == 0) launch_pair<A_MN, B_MN, EPI, 256>(g, st);
  else if constexpr (BN == 1) launch_pair<A_MN, B_MN, EPI, 128>(g, st);
  else launch_tc<BN, A_MN, B_MN, EPI>(g, st);
}

template <int BN>
void dispatch_bn(const GemmArgs& g, cudaStream_t st) {
  const bool amn = g.amaj == Major::MN, bmn = g.bmaj == Major::MN;
  switch (g.epi) {
    case Epi::Store:
      if (!amn && bmn) return run<BN, false, true, (int)Epi::Store>(g, st);
      if (!amn && !bmn) return run<BN, false, false, (int)Epi::Store>(g, st);
      break;
    case Epi::Bias:
      if (!amn && bmn) return run<BN, false, true, (int)Epi::Bias>(g, st);
      break;
    case Epi::BiasGelu:
      if (!amn && bmn) return run<BN, false, true, (int)Epi::BiasGelu>(g, st);
      break;
    case Epi::GeluBwd:
      if (!amn && !bmn) return run<BN, false, false, (int)Epi::GeluBwd>(g, st);
      break;
    case Epi::F32:
      if (amn && bmn) return run<BN, true, true, (int)Epi::F32>(g, st);
      break;
  }
  raise(3, "gemm_tc: unsupported operand majors for this epilogue");
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

bool gemm_tc_supported(const GemmArgs& g) {
  if (g.M < 1 || g.N < 32 || g.K < 1) return false;
  if (g.N % 32 != 0) return false;
  if (g.lda % 8 || g.ldb % 8 || g.ldc % 8) return false;
  if (!aligned16(g.A) || !aligned16(g.B) || !aligned16(g.C)) return false;
  for (int q = 0; q < g.a_shards; ++q)
    if (!aligned16(g.a_shard[q])) return false;
  for (int q = 0; q < g.b_shards; ++q)
    if (!aligned16(g.b_shard[q])) return false;
  if (g.epi == Epi::BiasGelu && !aligned16(g.C2)) return false;
  if (g.epi == Epi::GeluBwd && (g.ldaux % 8 || !aligned16(g.aux))) return false;
  const bool amn = g.amaj == Major::MN, bmn = g.bmaj == Major::MN;
  switch (g.epi) {
    case Epi::Store: return !amn;
    case Epi::Bias:
    case Epi::BiasGelu: return !amn && bmn;
    case Epi::GeluBwd: return !amn && !bmn;
    case Epi::F32: return amn && bmn;
  }
  return false;
}

// GEMMs with M, N >= 256 run on the CTA-pair kernel (measured 1443 vs 1350 TFLOP/s over the
// 22B layer's GEMMs); SPL_GEMM_PAIR=0 selects the single-CTA kernel for every shape.
static bool pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SPL_GEMM_PAIR");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

// Fraction of the CTA pairs' wave slots a tile grid fills (persistent kernel, 74 pairs).
static double wave_fill(int64_t tiles) {
  const int64_t pairs = kNumSMs / 2;
  const int64_t waves = (tiles + pairs - 1) / pairs;
  return (double)tiles / (double)(waves * pairs);
}
// SPL_GEMM_PAIR128=1 (A/B only): 256 x 128 pair tiles when they fill the last wave clearly
// better than 256 x 256 (the t > 1 shard widths: N = 768 at 22B t = 8 fills 65 % with
// 256-wide tiles, 86 % with 128). Measured slower: 22B t = 8 selective + SP per-GPU compute
// 2.79-2.87 -> 2.99-3.08 ms (the narrower tile's operand traffic outweighs the fuller wave).
static bool pair_narrow(const GemmArgs& g) {
  static const bool on = [] {
    const char* e = std::getenv("SPL_GEMM_PAIR128");
    return e != nullptr && e[0] == '1';
  }();
  if (!on) return false;
  const int64_t tm = (g.M + 255) / 256;
  return wave_fill(tm * ((g.N + 127) / 128)) > wave_fill(tm * ((g.N + 255) / 256)) + 0.05;
}

bool gemm_tc_pair_path(const GemmArgs& g) {
  return g.N >= 256 && g.M >= 256 && pair_enabled() && gemm_tc_supported(g);
}

void gemm_tc(const GemmArgs& g, cudaStream_t st) {
  if (g.a_shards > 1 || g.b_shards > 1)
    require(g.N >= 256 && g.M >= 256 && pair_enabled(), "sharded GEMM operands need the pair kernel");
  if (g.N >= 256 && g.M >= 256 && pair_enabled()) {
    if (pair_narrow(g)) dispatch_bn<1>(g, st);
    else dispatch_bn<0>(g, st);
  }
  else if (g.N >= 256) dispatch_bn<256>(g, st);
  else dispatch_bn<128>(g, st);
}

}  // namespace spl::k
