// Memory-bound kernels of the layer: LayerNorm fwd/bwd, fused bias-dropout-residual(+LN),
// dropout backward with bias-gradient column sums, parameter init, local-rank ordered sums.
//
// Design (HBM-bound): 16-byte vector loads/stores (8 bf16 / 4 fp32)
// when the row width allows, one CTA per row for row reductions with the row cached in
// registers, column-tiled CTAs (one 16-byte column vector per thread, a chunk of rows per
// CTA) for the column sums, fp32 statistics, deterministic two-level reductions.
#include <type_traits>

#include "kernels.hpp"
#include "rng_fast.cuh"

namespace spl::k {

namespace {

template <typename T, int VW>
__device__ __forceinline__ void load_vec(const T* __restrict__ p, float (&v)[VW]) {
  if constexpr (VW == 1) {
    v[0] = to_f(p[0]);
  } else if constexpr (std::is_same_v<T, float>) {
    static_assert(VW == 4, "fp32 vectors are float4");
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    static_assert(VW == 8, "bf16 vectors are 8 wide");
    const uint4 t = *reinterpret_cast<const uint4*>(p);
    const bf16* e = reinterpret_cast<const bf16*>(&t);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(e[i]);
  }
}

template <typename T, int VW>
__device__ __forceinline__ void store_vec(T* __restrict__ p, const float (&v)[VW]) {
  if constexpr (VW == 1) {
    p[0] = from_f<T>(v[0]);
  } else if constexpr (std::is_same_v<T, float>) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    uint4 t;
    bf16* e = reinterpret_cast<bf16*>(&t);
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = __float2bfloat16_rn(v[i]);
    *reinterpret_cast<uint4*>(p) = t;
  }
}

// round-trip through T so later math sees exactly the stored value
template <typename T>
__device__ __forceinline__ float round_t(float v) {
  if constexpr (std::is_same_v<T, float>) return v;
  else return __bfloat162float(__float2bfloat16_rn(v));
}

template <int VW>
__device__ __forceinline__ void store_mask(uint8_t* p, const uint8_t (&m)[VW]) {
  if constexpr (VW == 1) {
    p[0] = m[0];
  } else if constexpr (VW == 4) {
    *reinterpret_cast<uint32_t*>(p) =
        (uint32_t)m[0] | ((uint32_t)m[1] << 8) | ((uint32_t)m[2] << 16) | ((uint32_t)m[3] << 24);
  } else {
    uint2 t;
    t.x = (uint32_t)m[0] | ((uint32_t)m[1] << 8) | ((uint32_t)m[2] << 16) | ((uint32_t)m[3] << 24);
    t.y = (uint32_t)m[4] | ((uint32_t)m[5] << 8) | ((uint32_t)m[6] << 16) | ((uint32_t)m[7] << 24);
    *reinterpret_cast<uint2*>(p) = t;
  }
}

template <int VW>
__device__ __forceinline__ void load_mask(const uint8_t* p, uint8_t (&m)[VW]) {
  if constexpr (VW == 1) {
    m[0] = p[0];
  } else if constexpr (VW == 4) {
    const uint32_t t = *reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] = (uint8_t)(t >> (8 * i));
  } else {
    const uint2 t = *reinterpret_cast<const uint2*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      m[i] = (uint8_t)(t.x >> (8 * i));
      m[4 + i] = (uint8_t)(t.y >> (8 * i));
    }
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum over the CTA; every thread gets the result. `red` holds >= 32 floats.
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int nw = blockDim.x >> 5;
  if (nw == 1) return v;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = l < nw ? red[l] : 0.f;
  return warp_sum(t);
}

constexpr int kVPT = 8;  // vectors per thread for row-cached kernels

template <typename T>
constexpr int vec_width() {
  return 16 / sizeof(T);
}

// vectors per thread of the register-cached row kernels (0: too wide, generic kernel)
inline int pick_vpt(int64_t nvec) { return nvec <= 2048 ? 4 : (nvec <= 4096 ? 8 : 0); }
// threads for a register-cached row kernel: ceil(nvec / vpt) rounded up to whole warps
inline int vthreads(int64_t nvec, int vpt) {
  int64_t nt = (nvec + vpt - 1) / vpt;
  nt = ((nt + 31) / 32) * 32;
  return (int)std::max<int64_t>(32, nt);
}

inline int row_threads(int64_t nvec) {
  int64_t nt = (nvec + kVPT - 1) / kVPT;
  nt = ((nt + 31) / 32) * 32;
  if (nt < 32) nt = 32;
  return (int)nt;
}

// ---------------------------------------------------------------- LN forward
template <typename T, int VW>
__global__ void __launch_bounds__(512) ln_fwd_k(const T* __restrict__ x,
                                                const float* __restrict__ g,
                                                const float* __restrict__ b, T* __restrict__ y,
                                                float* __restrict__ mean,
                                                float* __restrict__ rstd, int h, float eps) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * h;
  T* yr = y + row * h;
  const int nvec = h / VW;
  float v[kVPT][VW];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kVPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
      load_vec<T, VW>(xr + vi * VW, v[i]);
#pragma unroll
      for (int j = 0; j < VW; ++j) s += v[i][j];
    }
  }
  const float mu = block_sum(s, red) / (float)h;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < kVPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
#pragma unroll
      for (int j = 0; j < VW; ++j) {
        const float d = v[i][j] - mu;
        q += d * d;
      }
    }
  }
  const float var = block_sum(q, red) / (float)h;
  const float rs = 1.0f / sqrtf(var + eps);
  if (threadIdx.x == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
#pragma unroll
  for (int i = 0; i < kVPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
      float o[VW];
#pragma unroll
      for (int j = 0; j < VW; ++j) {
        const int c = vi * VW + j;
        o[j] = (v[i][j] - mu) * rs * g[c] + b[c];
      }
      store_vec<T, VW>(yr + vi * VW, o);
    }
  }
}

// ---------------------------------------------------------------- bias-dropout-residual (+LN)
template <typename T, int VW, bool LN>
__global__ void __launch_bounds__(512) bdr_k(const T* __restrict__ a, const float* __restrict__ bias,
                                             const T* __restrict__ resid, T* __restrict__ r_out,
                                             uint8_t* __restrict__ mask_out, T* __restrict__ ln_out,
                                             const float* __restrict__ g,
                                             const float* __restrict__ lb, float* __restrict__ mean,
                                             float* __restrict__ rstd, int h, DropKey key,
                                             uint64_t base, float eps, int* nonfinite) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const int nvec = h / VW;
  float v[kVPT][VW];
  float s = 0.f;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < kVPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
      float av[VW], xv[VW];
      uint8_t m[VW];
      const int64_t off = row * h + (int64_t)vi * VW;
      load_vec<T, VW>(a + off, av);
      load_vec<T, VW>(resid + off, xv);
#pragma unroll
      for (int j = 0; j < VW; ++j) {
        const bool keep = drop_keep(key, base + (uint64_t)(off + j));
        m[j] = keep ? 1 : 0;
        const float t = (av[j] + bias[vi * VW + j]) * (keep ? 1.f : 0.f) * key.inv_keep;
        v[i][j] = round_t<T>(xv[j] + t);
        s += v[i][j];
        bad |= !isfinite(v[i][j]);
      }
      store_vec<T, VW>(r_out + off, v[i]);
      store_mask<VW>(mask_out + off, m);
    }
  }
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
  if constexpr (LN) {
    const float mu = block_sum(s, red) / (float)h;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < kVPT; ++i) {
      const int vi = threadIdx.x + i * blockDim.x;
      if (vi < nvec) {
#pragma unroll
        for (int j = 0; j < VW; ++j) {
          const float d = v[i][j] - mu;
          q += d * d;
        }
      }
    }
    const float var = block_sum(q, red) / (float)h;
    const float rs = 1.0f / sqrtf(var + eps);
    if (threadIdx.x == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
#pragma unroll
    for (int i = 0; i < kVPT; ++i) {
      const int vi = threadIdx.x + i * blockDim.x;
      if (vi < nvec) {
        float o[VW];
#pragma unroll
        for (int j = 0; j < VW; ++j) {
          const int c = vi * VW + j;
          o[j] = (v[i][j] - mu) * rs * g[c] + lb[c];
        }
        store_vec<T, VW>(ln_out + row * h + (int64_t)vi * VW, o);
      }
    }
  }
}

// ================================================================ register-cached row kernels
// One CTA per row; thread i owns the 16-byte vectors i, i+nt, ... (VPT of them, coalesced
// across the CTA) and keeps them *packed* in registers (4 regs per 8 bf16), so a row is read
// from HBM exactly once and the CTA stays small enough (≈40-64 regs) for full occupancy:
// nt = nvec/VPT threads <= 512: VPT = 4 up to 2048 vectors (192 threads at h = 6144),
// VPT = 8 up to 4096 (400 threads at h = 25600); wider rows take the generic kernels.
template <typename T>
constexpr int kVW = 16 / (int)sizeof(T);

template <typename T>
__device__ __forceinline__ void unpack(const uint4& r, float (&v)[kVW<T>]) {
  if constexpr (std::is_same_v<T, float>) {
    v[0] = __uint_as_float(r.x); v[1] = __uint_as_float(r.y);
    v[2] = __uint_as_float(r.z); v[3] = __uint_as_float(r.w);
  } else {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
}
template <typename T>
__device__ __forceinline__ uint4 pack(const float (&v)[kVW<T>]) {
  if constexpr (std::is_same_v<T, float>) {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                      __float_as_uint(v[3]));
  } else {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&b);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
}
__device__ __forceinline__ uint4 ld16(const void* p) {  // read-once data: no L1 allocation
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st16(void* p, const uint4& v) {
  *reinterpret_cast<uint4*>(p) = v;
}
// fp32 per-column parameters (gain / bias): VW of them at column c (16-byte aligned)
template <int VW>
__device__ __forceinline__ void ldcols(const float* __restrict__ p, int c, float (&v)[VW]) {
#pragma unroll
  for (int i = 0; i < VW; i += 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p + c + i));
    v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
  }
}
// Both sums over the CTA in one pass (one pair of barriers); `red` holds >= 64 floats.
__device__ __forceinline__ float2 block_sum2(float a, float b, float* red) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int nw = blockDim.x >> 5;
  if (nw == 1) return make_float2(a, b);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    red[w] = a;
    red[32 + w] = b;
  }
  __syncthreads();
  a = l < nw ? red[l] : 0.f;
  b = l < nw ? red[32 + l] : 0.f;
  return make_float2(warp_sum(a), warp_sum(b));
}

template <typename T, int VPT>
__global__ void __launch_bounds__(512) ln_fwd_v(const T* __restrict__ x,
                                                 const float* __restrict__ g,
                                                 const float* __restrict__ b, T* __restrict__ y,
                                                 float* __restrict__ mean,
                                                 float* __restrict__ rstd, int h, float eps) {
  constexpr int VW = kVW<T>;
  __shared__ float red[64];
  const int64_t row = blockIdx.x;
  const int nvec = h / VW;
  uint4 raw[VPT];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) raw[i] = ld16(x + row * h + (int64_t)vi * VW);
  }
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    if (threadIdx.x + i * blockDim.x < nvec) {
      float v[VW];
      unpack<T>(raw[i], v);
#pragma unroll
      for (int j = 0; j < VW; ++j) s += v[j];
    }
  }
  const float mu = block_sum(s, red) / (float)h;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    if (threadIdx.x + i * blockDim.x < nvec) {
      float v[VW];
      unpack<T>(raw[i], v);
#pragma unroll
      for (int j = 0; j < VW; ++j) q += (v[j] - mu) * (v[j] - mu);
    }
  }
  const float var = block_sum(q, red) / (float)h;
  const float rs = 1.0f / sqrtf(var + eps);
  if (threadIdx.x == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
      float v[VW], gv[VW], bv[VW], o[VW];
      unpack<T>(raw[i], v);
      ldcols<VW>(g, vi * VW, gv);
      ldcols<VW>(b, vi * VW, bv);
#pragma unroll
      for (int j = 0; j < VW; ++j) o[j] = (v[j] - mu) * rs * gv[j] + bv[j];
      st16(y + row * h + (int64_t)vi * VW, pack<T>(o));
    }
  }
}

// ---- fused reduce-scatter consumer: slots landed by peers (or simulated ranks)
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// every source has signalled past this rank's generation (thread 0 polls, the CTA waits)
__device__ __forceinline__ void wait_slots(const SlotSrc& a) {
  if (a.flags == nullptr) return;
  if (threadIdx.x == 0) {
    const uint32_t target = ld_acquire_sys(a.gen) + 1u;
    for (int q = 0; q < a.n; ++q)
      while ((int32_t)(ld_acquire_sys(a.flags + q) - target) < 0) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}
__device__ __forceinline__ uint4 ld16_coherent(const void* p) {  // data landed by a peer (L2)
  uint4 r;
  asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// rank-ordered fp32 sum of the slots at element offset `off`, rounded to T (as rs_local_k)
template <typename T>
__device__ __forceinline__ uint4 sum_slots(const SlotSrc& a, int64_t off) {
  constexpr int VW = kVW<T>;
  float acc[VW], v[VW];
  unpack<T>(ld16_coherent(static_cast<const T*>(a.p[0]) + off), acc);
  for (int q = 1; q < a.n; ++q) {
    unpack<T>(ld16_coherent(static_cast<const T*>(a.p[q]) + off), v);
#pragma unroll
    for (int j = 0; j < VW; ++j) acc[j] += v[j];
  }
  return pack<T>(acc);
}

__global__ void p2p_signal_k(FlagPtrs f) {
  __threadfence_system();  // this rank's landed rows (previous kernel) before the counters
  if ((int)threadIdx.x < f.n)
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(f.p[threadIdx.x]) : "memory");
}
__global__ void p2p_advance_k(uint32_t* gen) { *gen += 1u; }

template <typename T>
__global__ void reduce_slots_k(SlotSrc a, T* __restrict__ out, int64_t nvec) {
  wait_slots(a);
  constexpr int VW = kVW<T>;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x)
    st16(out + i * VW, sum_slots<T>(a, i * VW));
}

// Bias + dropout + residual (+ LayerNorm of the result). The dropout keep bits of the VW
// elements of a vector come from the counter RNG in its hot-loop form (rng_fast.cuh): the
// high half of the 64-bit counter is shared by the vector unless its low half carries.
// SL: the input partial is the rank-ordered sum of the fused reduce-scatter's landing slots.
template <typename T, int VPT, bool LN, bool SL>
__global__ void __launch_bounds__(512) bdr_v(const T* __restrict__ a, SlotSrc slots,
                                              const float* __restrict__ bias,
                                              const T* __restrict__ resid, T* __restrict__ r_out,
                                              uint8_t* __restrict__ mask_out,
                                              T* __restrict__ ln_out, const float* __restrict__ g,
                                              const float* __restrict__ lb,
                                              float* __restrict__ mean, float* __restrict__ rstd,
                                              int h, DropKey key, uint64_t base, float eps,
                                              int* nonfinite, rngk::ShiftMuls sm) {
  using namespace rngk;
  constexpr int VW = kVW<T>;
  __shared__ float red[64];
  const int64_t row = blockIdx.x;
  const int nvec = h / VW;
  const uint64_t tsh = key.thresh << 11;
  const uint32_t mixed_lo = (uint32_t)key.mixed, mixed_hi = (uint32_t)(key.mixed >> 32);
  const uint32_t t_lo = (uint32_t)tsh, t_hi = (uint32_t)(tsh >> 32);
  uint4 ar[VPT], xr[VPT];
  if constexpr (SL) wait_slots(slots);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
      const int64_t off = row * h + (int64_t)vi * VW;
      if constexpr (SL) ar[i] = sum_slots<T>(slots, off);
      else ar[i] = ld16(a + off);
      xr[i] = ld16(resid + off);
    }
  }
  float s = 0.f;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
      const int64_t off = row * h + (int64_t)vi * VW;
      uint32_t kb = (1u << VW) - 1u;
      if (key.thresh != 0) {
        const uint64_t B = base + (uint64_t)off + kC + kG;
        const uint32_t blo = (uint32_t)B, bhi = (uint32_t)(B >> 32);
        kb = 0;
        if (blo <= 0xffffffffu - (uint32_t)(VW - 1)) {
          const uint32_t hx = bhi ^ (bhi >> 30);
          const uint32_t hc = hx * 0x1ce4e5b9u;
          // fast form (as keep_bits_k): lo >> 30 constant over the VW keys, keep decided on the
          // raw high word; a key near the threshold (or a 2^30 crossing) takes the exact form
          bool rare = (blo >> 30) != ((blo + (uint32_t)(VW - 1)) >> 30);
          if (!rare) {
            const uint32_t c30 = __funnelshift_r(blo, bhi, 30);
            const uint32_t t_even = t_hi & ~1u;
#pragma unroll
            for (int j = 0; j < VW; ++j) {
              const uint32_t raw = hash_hi<true, true>(blo + j, bhi, hc, mixed_lo, mixed_hi, sm, c30);
              if (raw > t_hi) kb |= 1u << j;
              rare |= raw - t_even < 2u;
            }
          }
          if (rare) {
            kb = 0;
#pragma unroll 1
            for (int j = 0; j < VW; ++j)
              if (keep_fast(blo + j, bhi, hc, hx, mixed_lo, mixed_hi, t_lo, t_hi, sm)) kb |= 1u << j;
          }
        } else {
          for (int j = 0; j < VW; ++j)
            if (mix_post((mix_post(B + j) ^ key.mixed) + kG) >= tsh) kb |= 1u << j;
        }
      }
      float av[VW], xv[VW], bv[VW], v[VW];
      unpack<T>(ar[i], av);
      unpack<T>(xr[i], xv);
      ldcols<VW>(bias, vi * VW, bv);
      uint32_t mw[2] = {0u, 0u};
#pragma unroll
      for (int j = 0; j < VW; ++j) {
        const bool keep = (kb >> j) & 1u;
        const float t = (av[j] + bv[j]) * (keep ? 1.f : 0.f) * key.inv_keep;
        v[j] = round_t<T>(xv[j] + t);
        s += v[j];
        bad |= !isfinite(v[j]);
        mw[j >> 2] |= (keep ? 1u : 0u) << (8 * (j & 3));
      }
      xr[i] = pack<T>(v);  // the residual output, exact in T
      st16(r_out + off, xr[i]);
      if constexpr (VW == 8) *reinterpret_cast<uint2*>(mask_out + off) = make_uint2(mw[0], mw[1]);
      else *reinterpret_cast<uint32_t*>(mask_out + off) = mw[0];
    }
  }
  if (nonfinite != nullptr && bad) atomicOr(nonfinite, 1);
  if constexpr (LN) {
    const float mu = block_sum(s, red) / (float)h;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      if (threadIdx.x + i * blockDim.x < nvec) {
        float v[VW];
        unpack<T>(xr[i], v);
#pragma unroll
        for (int j = 0; j < VW; ++j) q += (v[j] - mu) * (v[j] - mu);
      }
    }
    const float var = block_sum(q, red) / (float)h;
    const float rs = 1.0f / sqrtf(var + eps);
    if (threadIdx.x == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int vi = threadIdx.x + i * blockDim.x;
      if (vi < nvec) {
        float v[VW], gv[VW], bv[VW], o[VW];
        unpack<T>(xr[i], v);
        ldcols<VW>(g, vi * VW, gv);
        ldcols<VW>(lb, vi * VW, bv);
#pragma unroll
        for (int j = 0; j < VW; ++j) o[j] = (v[j] - mu) * rs * gv[j] + bv[j];
        st16(ln_out + row * h + (int64_t)vi * VW, pack<T>(o));
      }
    }
  }
}

// LN backward, dx part: dx = resid + rs·(dŷ - mean(dŷ) - x̂·mean(dŷ·x̂)), dŷ = dy·γ; dy, x
// and resid each read once (packed in registers), one two-value CTA reduction.
template <typename T, int VPT>
__global__ void __launch_bounds__(512) ln_bwd_dx_v(const T* __restrict__ dy, const T* __restrict__ x,
                                                   const float* __restrict__ mean,
                                                   const float* __restrict__ rstd,
                                                   const float* __restrict__ g,
                                                   const T* __restrict__ resid,
                                                   T* __restrict__ dx, int h) {
  constexpr int VW = kVW<T>;
  __shared__ float red[64];
  const int64_t row = blockIdx.x;
  const int nvec = h / VW;
  uint4 dr[VPT], xr[VPT], rr[VPT];
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
      const int64_t off = row * h + (int64_t)vi * VW;
      dr[i] = ld16(dy + off);
      xr[i] = ld16(x + off);
      rr[i] = ld16(resid + off);
    }
  }
  const float mu = mean[row], rs = rstd[row];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
      float dv[VW], xv[VW], gv[VW];
      unpack<T>(dr[i], dv);
      unpack<T>(xr[i], xv);
      ldcols<VW>(g, vi * VW, gv);
#pragma unroll
      for (int j = 0; j < VW; ++j) {
        const float xhat = (xv[j] - mu) * rs;
        const float dxhat = dv[j] * gv[j];
        s1 += dxhat;
        s2 += dxhat * xhat;
      }
    }
  }
  const float2 ss = block_sum2(s1, s2, red);
  const float inv_h = 1.0f / (float)h;
  const float m1 = ss.x * inv_h, m2 = ss.y * inv_h;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int vi = threadIdx.x + i * blockDim.x;
    if (vi < nvec) {
      float dv[VW], xv[VW], rv[VW], gv[VW], o[VW];
      unpack<T>(dr[i], dv);
      unpack<T>(xr[i], xv);
      unpack<T>(rr[i], rv);
      ldcols<VW>(g, vi * VW, gv);
#pragma unroll
      for (int j = 0; j < VW; ++j) {
        const float xhat = (xv[j] - mu) * rs;
        o[j] = rv[j] + rs * (dv[j] * gv[j] - m1 - xhat * m2);
      }
      st16(dx + row * h + (int64_t)vi * VW, pack<T>(o));
    }
  }
}

// ---------------------------------------------------------------- LN backward, dx part
// Row per CTA; two passes over the row (the second hits L1/L2), no column accumulation.
template <typename T, int VW>
__global__ void __launch_bounds__(512) ln_bwd_dx_k(const T* __restrict__ dy, const T* __restrict__ x,
                                                  const float* __restrict__ mean,
                                                  const float* __restrict__ rstd,
                                                  const float* __restrict__ g,
                                                  const T* __restrict__ resid,
                                                  T* __restrict__ dx, int h) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const int nvec = h / VW;
  const float mu = mean[row], rs = rstd[row];
  float s1 = 0.f, s2 = 0.f;
  for (int vi = threadIdx.x; vi < nvec; vi += blockDim.x) {
    float dv[VW], xv[VW];
    load_vec<T, VW>(dy + row * h + (int64_t)vi * VW, dv);
    load_vec<T, VW>(x + row * h + (int64_t)vi * VW, xv);
#pragma unroll
    for (int j = 0; j < VW; ++j) {
      const float xhat = (xv[j] - mu) * rs;
      const float dxhat = dv[j] * g[vi * VW + j];
      s1 += dxhat;
      s2 += dxhat * xhat;
    }
  }
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  const float inv_h = 1.0f / (float)h;
  for (int vi = threadIdx.x; vi < nvec; vi += blockDim.x) {
    float dv[VW], xv[VW], rv[VW], o[VW];
    const int64_t off = row * h + (int64_t)vi * VW;
    load_vec<T, VW>(dy + off, dv);
    load_vec<T, VW>(x + off, xv);
    load_vec<T, VW>(resid + off, rv);
#pragma unroll
    for (int j = 0; j < VW; ++j) {
      const float xhat = (xv[j] - mu) * rs;
      const float dxhat = dv[j] * g[vi * VW + j];
      o[j] = rv[j] + rs * (dxhat - inv_h * s1 - xhat * inv_h * s2);
    }
    store_vec<T, VW>(dx + off, o);
  }
}

// ---------------------------------------------------------------- column-tiled kernels
// LN gain/bias partial gradients: pg[c][j] = sum dy*xhat, pb[c][j] = sum dy over chunk rows.
template <typename T, int VW>
__global__ void ln_bwd_params_k(const T* __restrict__ dy, const T* __restrict__ x,
                                const float* __restrict__ mean, const float* __restrict__ rstd,
                                float* __restrict__ pg, float* __restrict__ pb, int64_t rows,
                                int h, int chunk) {
  const int vi = blockIdx.x * blockDim.x + threadIdx.x;
  if (vi * VW >= h) return;
  const int64_t r0 = (int64_t)blockIdx.y * chunk;
  const int64_t r1 = min(rows, r0 + chunk);
  float ag[VW], ab[VW];
#pragma unroll
  for (int j = 0; j < VW; ++j) ag[j] = ab[j] = 0.f;
#pragma unroll 8
  for (int64_t r = r0; r < r1; ++r) {
    float dv[VW], xv[VW];
    load_vec<T, VW>(dy + r * h + (int64_t)vi * VW, dv);
    load_vec<T, VW>(x + r * h + (int64_t)vi * VW, xv);
    const float mu = mean[r], rs = rstd[r];
#pragma unroll
    for (int j = 0; j < VW; ++j) {
      ag[j] += dv[j] * ((xv[j] - mu) * rs);
      ab[j] += dv[j];
    }
  }
  float* og = pg + (int64_t)blockIdx.y * h + vi * VW;
  float* ob = pb + (int64_t)blockIdx.y * h + vi * VW;
#pragma unroll
  for (int j = 0; j < VW; ++j) {
    og[j] = ag[j];
    ob[j] = ab[j];
  }
}

template <typename T, int VW>
__global__ void dropout_bwd_colsum_k(const T* __restrict__ dy, const uint8_t* __restrict__ mask,
                                     float inv_keep, T* __restrict__ out,
                                     float* __restrict__ partials, int64_t rows, int h,
                                     int chunk) {
  const int vi = blockIdx.x * blockDim.x + threadIdx.x;
  if (vi * VW >= h) return;
  const int64_t r0 = (int64_t)blockIdx.y * chunk;
  const int64_t r1 = min(rows, r0 + chunk);
  float acc[VW];
#pragma unroll
  for (int j = 0; j < VW; ++j) acc[j] = 0.f;
#pragma unroll 8
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t off = r * h + (int64_t)vi * VW;
    float dv[VW], o[VW];
    uint8_t m[VW];
    load_vec<T, VW>(dy + off, dv);
    load_mask<VW>(mask + off, m);
#pragma unroll
    for (int j = 0; j < VW; ++j) {
      o[j] = dv[j] * (float)m[j] * inv_keep;
      acc[j] += o[j];
    }
    store_vec<T, VW>(out + off, o);
  }
  float* p = partials + (int64_t)blockIdx.y * h + vi * VW;
#pragma unroll
  for (int j = 0; j < VW; ++j) p[j] = acc[j];
}

// 16-byte column vectors (VW columns per thread), a chunk of rows per CTA row
template <typename T>
__global__ void colsum_partial_v(const T* __restrict__ x, int64_t rows, int64_t n, int64_t ld,
                                 float* __restrict__ partials, int chunk) {
  constexpr int VW = kVW<T>;
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VW;
  if (c >= n) return;
  const int64_t r0 = (int64_t)blockIdx.y * chunk;
  const int64_t r1 = min(rows, r0 + chunk);
  float acc[VW];
#pragma unroll
  for (int j = 0; j < VW; ++j) acc[j] = 0.f;
#pragma unroll 4
  for (int64_t r = r0; r < r1; ++r) {
    float v[VW];
    unpack<T>(ld16(x + r * ld + c), v);
#pragma unroll
    for (int j = 0; j < VW; ++j) acc[j] += v[j];
  }
  float* p = partials + (int64_t)blockIdx.y * n + c;
#pragma unroll
  for (int j = 0; j < VW; j += 4)
    *reinterpret_cast<float4*>(p + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
}

template <typename T>
__global__ void colsum_partial_k(const T* __restrict__ x, int64_t rows, int64_t n, int64_t ld,
                                 float* __restrict__ partials, int chunk) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t r0 = (int64_t)blockIdx.y * chunk;
  const int64_t r1 = min(rows, r0 + chunk);
  float acc = 0.f;
  for (int64_t r = r0; r < r1; ++r) acc += to_f(x[r * ld + j]);
  partials[(int64_t)blockIdx.y * n + j] = acc;
}

// out[j] (+)= sum_c partials[c][j]. CTA = 32 columns x 8 chunk groups: every thread sums its
// group's chunks with all loads in flight, then the 8 group sums are added in a fixed order
// (deterministic; the chunk count is ~rows/64, so a column is far too short to stream alone).
__global__ void __launch_bounds__(256) reduce_partials_k(const float* __restrict__ partials,
                                                         int nchunks, int64_t n,
                                                         float* __restrict__ out, int accumulate) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  float acc = 0.f;
  if (j < n) {
    const int per = (nchunks + 7) / 8;
    const int c0 = grp * per, c1 = min(nchunks, c0 + per);
#pragma unroll 8
    for (int c = c0; c < c1; ++c) acc += partials[(int64_t)c * n + j];
  }
  red[grp][lane] = acc;
  __syncthreads();
  if (grp == 0 && j < n) {
    float t = red[0][lane];
#pragma unroll
    for (int g = 1; g < 8; ++g) t += red[g][lane];
    out[j] = accumulate ? out[j] + t : t;
  }
}

// ---------------------------------------------------------------- init
template <typename T>
__device__ __forceinline__ T from_d(double v);
template <>
__device__ __forceinline__ float from_d<float>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ bf16 from_d<bf16>(double v) { return __double2bfloat16(v); }

template <typename T>
__global__ void init_uniform_k(T* __restrict__ out, int64_t rows, int64_t cols, int64_t ld_out,
                               int64_t row0, int64_t col0, int64_t ld_full, uint64_t key,
                               double lo, double hi, double add) {
  const int64_t n = rows * cols;
  const double span = __dsub_rn(hi, lo);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / cols, j = t % cols;
    const uint64_t g = (uint64_t)((row0 + i) * ld_full + col0 + j);
    const double u = (double)(hash_counter(key, g) >> 11) * 0x1.0p-53;
    double v = __dadd_rn(lo, __dmul_rn(span, u));
    if (add != 0.0) v = __dadd_rn(v, add);
    out[i * ld_out + j] = from_d<T>(v);
  }
}

// ---------------------------------------------------------------- ordered sums / casts
template <typename T>
__global__ void ordered_sum_k(const T* const* __restrict__ parts, int nparts, int64_t offset,
                              int64_t n, T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = to_f(parts[0][offset + i]);
    for (int r = 1; r < nparts; ++r) acc += to_f(parts[r][offset + i]);
    out[i] = from_f<T>(acc);
  }
}

__global__ void ordered_sum_f32_k(const float* const* __restrict__ parts, int nparts, int64_t n,
                                  float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = parts[0][i];
    for (int r = 1; r < nparts; ++r) acc += parts[r][i];
    out[i] = acc;
  }
}

template <typename T>
__global__ void cast_f64_k(const T* __restrict__ in, double* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)to_f(in[i]);
}

__global__ void u8_f64_k(const uint8_t* __restrict__ in, double* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i];
}

inline int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > kNumSMs * 32) g = kNumSMs * 32;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

// ====================================================================== launchers
template <typename T>
void init_uniform(T* out, int64_t rows, int64_t cols, int64_t ld_out, int64_t row0,
                  int64_t col0, int64_t ld_full, uint64_t key, double lo, double hi, double add,
                  cudaStream_t st) {
  const int64_t n = rows * cols;
  if (n == 0) return;
  init_uniform_k<T><<<grid_for(n, 256), 256, 0, st>>>(out, rows, cols, ld_out, row0, col0,
                                                      ld_full, key, lo, hi, add);
  SPL_CHECK_LAUNCH();
}

template <typename T>
void layernorm_fwd(const T* x, const float* gain, const float* bias, T* y, float* mean,
                   float* rstd, int64_t rows, int64_t h, float eps, cudaStream_t st) {
  if (rows == 0) return;
  constexpr int VW = vec_width<T>();
  if (h % VW == 0 && pick_vpt(h / VW) == 4) {
    ln_fwd_v<T, 4><<<(unsigned)rows, vthreads(h / VW, 4), 0, st>>>(x, gain, bias, y, mean, rstd,
                                                                   (int)h, eps);
  } else if (h % VW == 0 && pick_vpt(h / VW) == 8) {
    ln_fwd_v<T, 8><<<(unsigned)rows, vthreads(h / VW, 8), 0, st>>>(x, gain, bias, y, mean, rstd,
                                                                   (int)h, eps);
  } else {
    require(h <= 512 * kVPT, "layernorm: hidden too large for the unaligned path");
    ln_fwd_k<T, 1><<<(unsigned)rows, row_threads(h), 0, st>>>(x, gain, bias, y, mean, rstd,
                                                              (int)h, eps);
  }
  SPL_CHECK_LAUNCH();
}

template <typename T>
void bias_dropout_residual(const T* a, const float* bias, const T* resid, T* r_out,
                           uint8_t* mask_out, T* ln_out, const float* gain, const float* lnb,
                           float* mean, float* rstd, int64_t rows, int64_t h, DropKey key,
                           uint64_t base_index, float eps, int* nonfinite, cudaStream_t st) {
  if (rows == 0) return;
  constexpr int VW = vec_width<T>();
  if (h % VW == 0 && pick_vpt(h / VW) != 0) {
    const rngk::ShiftMuls sm{4u, 32u, 2u, 1u};
    const int vpt = pick_vpt(h / VW);
    const unsigned nt = (unsigned)vthreads(h / VW, vpt);
#define SPL_BDRV(VPTX, LNX)                                                                   \
  bdr_v<T, VPTX, LNX, false><<<(unsigned)rows, nt, 0, st>>>(a, SlotSrc{}, bias, resid, r_out, \
                                                     mask_out, ln_out, gain, lnb, mean, rstd, \
                                                     (int)h, key, base_index, eps, nonfinite, sm)
    if (vpt == 4) {
      if (ln_out) SPL_BDRV(4, true); else SPL_BDRV(4, false);
    } else {
      if (ln_out) SPL_BDRV(8, true); else SPL_BDRV(8, false);
    }
#undef SPL_BDRV
    SPL_CHECK_LAUNCH();
    return;
  }
  const bool vec = false;
  require(h <= 512 * kVPT, "bias_dropout_residual: hidden too large");
  const int nt = row_threads(vec ? h / VW : h);
#define SPL_BDR(VWX, LNX)                                                                    \
  bdr_k<T, VWX, LNX><<<(unsigned)rows, nt, 0, st>>>(a, bias, resid, r_out, mask_out, ln_out, \
                                                    gain, lnb, mean, rstd, (int)h, key,      \
                                                    base_index, eps, nonfinite)
  if (vec) {
    if (ln_out) SPL_BDR(VW, true); else SPL_BDR(VW, false);
  } else {
    if (ln_out) SPL_BDR(1, true); else SPL_BDR(1, false);
  }
#undef SPL_BDR
  SPL_CHECK_LAUNCH();
}

void p2p_signal(const FlagPtrs& f, cudaStream_t st) {
  require(f.n >= 1 && f.n <= kMaxScatterRanks, "p2p_signal: bad rank count");
  p2p_signal_k<<<1, 32, 0, st>>>(f);
  SPL_CHECK_LAUNCH();
}
void p2p_advance(uint32_t* gen, cudaStream_t st) {
  p2p_advance_k<<<1, 1, 0, st>>>(gen);
  SPL_CHECK_LAUNCH();
}

template <typename T>
void bias_dropout_residual_slots(const SlotSrc& a, const float* bias, const T* resid, T* r_out,
                                 uint8_t* mask_out, T* ln_out, const float* gain, const float* lnb,
                                 float* mean, float* rstd, int64_t rows, int64_t h, DropKey key,
                                 uint64_t base_index, float eps, int* nonfinite, cudaStream_t st) {
  if (rows == 0) return;
  constexpr int VW = vec_width<T>();
  require(h % VW == 0 && pick_vpt(h / VW) != 0 && a.n >= 1,
          "fused reduce-scatter consumer: hidden must be a multiple of the vector width");
  const rngk::ShiftMuls sm{4u, 32u, 2u, 1u};
  const int vpt = pick_vpt(h / VW);
  const unsigned nt = (unsigned)vthreads(h / VW, vpt);
#define SPL_BDRS(VPTX, LNX)                                                                    \
  bdr_v<T, VPTX, LNX, true><<<(unsigned)rows, nt, 0, st>>>(nullptr, a, bias, resid, r_out,      \
                                                           mask_out, ln_out, gain, lnb, mean,  \
                                                           rstd, (int)h, key, base_index, eps, \
                                                           nonfinite, sm)
  if (vpt == 4) {
    if (ln_out) SPL_BDRS(4, true); else SPL_BDRS(4, false);
  } else {
    if (ln_out) SPL_BDRS(8, true); else SPL_BDRS(8, false);
  }
#undef SPL_BDRS
  SPL_CHECK_LAUNCH();
}

template <typename T>
void reduce_slots(const SlotSrc& a, T* out, int64_t n, cudaStream_t st) {
  constexpr int VW = vec_width<T>();
  require(n % VW == 0 && a.n >= 1, "reduce_slots: size must be a multiple of the vector width");
  const int64_t nvec = n / VW;
  reduce_slots_k<T><<<grid_for(nvec, 256), 256, 0, st>>>(a, out, nvec);
  SPL_CHECK_LAUNCH();
}

template <typename T>
void dropout_bwd_colsum(const T* dy, const uint8_t* mask, float inv_keep, T* out,
                        float* partials, int64_t rows, int64_t h, int chunk_rows,
                        cudaStream_t st) {
  if (rows == 0) return;
  constexpr int VW = vec_width<T>();
  const int nch = num_chunks(rows, chunk_rows);
  if (h % VW == 0) {
    const int64_t nvec = h / VW;
    dim3 grid((unsigned)((nvec + 127) / 128), (unsigned)nch);
    dropout_bwd_colsum_k<T, VW><<<grid, 128, 0, st>>>(dy, mask, inv_keep, out, partials, rows,
                                                      (int)h, chunk_rows);
  } else {
    dim3 grid((unsigned)((h + 127) / 128), (unsigned)nch);
    dropout_bwd_colsum_k<T, 1><<<grid, 128, 0, st>>>(dy, mask, inv_keep, out, partials, rows,
                                                     (int)h, chunk_rows);
  }
  SPL_CHECK_LAUNCH();
}

template <typename T>
void layernorm_bwd(const T* dy, const T* x, const float* mean, const float* rstd,
                   const float* gain, const T* resid_grad, T* dx, float* pgain, float* pbias,
                   int64_t rows, int64_t h, int chunk_rows, cudaStream_t st) {
  if (rows == 0) return;
  constexpr int VW = vec_width<T>();
  const int nch = num_chunks(rows, chunk_rows);
  if (h % VW == 0) {
    const int64_t nvec = h / VW;
    if (pick_vpt(nvec) == 4) {
      ln_bwd_dx_v<T, 4><<<(unsigned)rows, vthreads(nvec, 4), 0, st>>>(dy, x, mean, rstd, gain,
                                                                      resid_grad, dx, (int)h);
    } else if (pick_vpt(nvec) == 8) {
      ln_bwd_dx_v<T, 8><<<(unsigned)rows, vthreads(nvec, 8), 0, st>>>(dy, x, mean, rstd, gain,
                                                                      resid_grad, dx, (int)h);
    } else {
      int nt = (int)std::min<int64_t>(512, ((nvec + 31) / 32) * 32);
      ln_bwd_dx_k<T, VW><<<(unsigned)rows, nt, 0, st>>>(dy, x, mean, rstd, gain, resid_grad, dx,
                                                        (int)h);
    }
    dim3 grid((unsigned)((nvec + 127) / 128), (unsigned)nch);
    ln_bwd_params_k<T, VW><<<grid, 128, 0, st>>>(dy, x, mean, rstd, pgain, pbias, rows, (int)h,
                                                 chunk_rows);
  } else {
    int nt = (int)std::min<int64_t>(512, ((h + 31) / 32) * 32);
    ln_bwd_dx_k<T, 1><<<(unsigned)rows, nt, 0, st>>>(dy, x, mean, rstd, gain, resid_grad, dx,
                                                     (int)h);
    dim3 grid((unsigned)((h + 127) / 128), (unsigned)nch);
    ln_bwd_params_k<T, 1><<<grid, 128, 0, st>>>(dy, x, mean, rstd, pgain, pbias, rows, (int)h,
                                                chunk_rows);
  }
  SPL_CHECK_LAUNCH();
}

template <typename T>
void colsum_partial(const T* x, int64_t rows, int64_t n, int64_t ld, float* partials,
                    int chunk_rows, cudaStream_t st) {
  if (rows == 0 || n == 0) return;
  constexpr int VW = vec_width<T>();
  if (n % VW == 0 && ld % VW == 0 && ((uintptr_t)x & 15) == 0) {
    dim3 grid((unsigned)((n / VW + 127) / 128), (unsigned)num_chunks(rows, chunk_rows));
    colsum_partial_v<T><<<grid, 128, 0, st>>>(x, rows, n, ld, partials, chunk_rows);
  } else {
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)num_chunks(rows, chunk_rows));
    colsum_partial_k<T><<<grid, 128, 0, st>>>(x, rows, n, ld, partials, chunk_rows);
  }
  SPL_CHECK_LAUNCH();
}

void reduce_partials(const float* partials, int nchunks, int64_t n, float* out, bool accumulate,
                     cudaStream_t st) {
  if (n == 0) return;
  reduce_partials_k<<<(unsigned)((n + 31) / 32), 256, 0, st>>>(partials, nchunks, n, out,
                                                               accumulate ? 1 : 0);
  SPL_CHECK_LAUNCH();
}

template <typename T>
void ordered_sum(const T* const* parts_dev, int nparts, int64_t offset, int64_t n, T* out,
                 cudaStream_t st) {
  if (n == 0) return;
  ordered_sum_k<T><<<grid_for(n, 256), 256, 0, st>>>(parts_dev, nparts, offset, n, out);
  SPL_CHECK_LAUNCH();
}

void ordered_sum_f32(const float* const* parts_dev, int nparts, int64_t n, float* out,
                     cudaStream_t st) {
  if (n == 0) return;
  ordered_sum_f32_k<<<grid_for(n, 256), 256, 0, st>>>(parts_dev, nparts, n, out);
  SPL_CHECK_LAUNCH();
}

template <typename T>
void cast_to_f64(const T* in, double* out, int64_t n, cudaStream_t st) {
  if (n == 0) return;
  cast_f64_k<T><<<grid_for(n, 256), 256, 0, st>>>(in, out, n);
  SPL_CHECK_LAUNCH();
}

void u8_to_f64(const uint8_t* in, double* out, int64_t n, cudaStream_t st) {
  if (n == 0) return;
  u8_f64_k<<<grid_for(n, 256), 256, 0, st>>>(in, out, n);
  SPL_CHECK_LAUNCH();
}

void f32_to_f64(const float* in, double* out, int64_t n, cudaStream_t st) {
  cast_to_f64<float>(in, out, n, st);
}

#define SPL_INST(T)                                                                           \
  template void init_uniform<T>(T*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,     \
                                uint64_t, double, double, double, cudaStream_t);             \
  template void layernorm_fwd<T>(const T*, const float*, const float*, T*, float*, float*,   \
                                 int64_t, int64_t, float, cudaStream_t);                     \
  template void bias_dropout_residual_slots<T>(const SlotSrc&, const float*, const T*, T*,    \
                                               uint8_t*, T*, const float*, const float*,      \
                                               float*, float*, int64_t, int64_t, DropKey,     \
                                               uint64_t, float, int*, cudaStream_t);          \
  template void reduce_slots<T>(const SlotSrc&, T*, int64_t, cudaStream_t);                   \
  template void bias_dropout_residual<T>(const T*, const float*, const T*, T*, uint8_t*, T*,  \
                                         const float*, const float*, float*, float*, int64_t, \
                                         int64_t, DropKey, uint64_t, float, int*,             \
                                         cudaStream_t);                                       \
  template void dropout_bwd_colsum<T>(const T*, const uint8_t*, float, T*, float*, int64_t,  \
                                      int64_t, int, cudaStream_t);                            \
  template void layernorm_bwd<T>(const T*, const T*, const float*, const float*,             \
                                 const float*, const T*, T*, float*, float*, int64_t,        \
                                 int64_t, int, cudaStream_t);                                 \
  template void colsum_partial<T>(const T*, int64_t, int64_t, int64_t, float*, int,           \
                                  cudaStream_t);                                              \
  template void ordered_sum<T>(const T* const*, int, int64_t, int64_t, T*, cudaStream_t);    \
  template void cast_to_f64<T>(const T*, double*, int64_t, cudaStream_t);
SPL_INST(float)
SPL_INST(bf16)
#undef SPL_INST

}  // namespace spl::k
