// Memory-bound kernels of the layer: LayerNorm fwd/bwd, fused bias-dropout-residual(+LN),
// dropout backward with bias-gradient column sums, parameter init, local-rank ordered sums.
//
// Design (HBM-bound): 16-byte vector loads/stores (8 bf16 / 4 fp32)
// when the row width allows, one CTA per row for row reductions with the row cached in
// registers, column-tiled CTAs (one 16-byte column vector per thread, a chunk of rows per
// CTA) for the column sums, fp32 statistics, deterministic two-level reductions.
#include <type_traits>

#include "kernels.hpp"

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

__global__ void reduce_partials_k(const float* __restrict__ partials, int nchunks, int64_t n,
                                  float* __restrict__ out, int accumulate) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float acc = accumulate ? out[j] : 0.f;
  for (int c = 0; c < nchunks; ++c) acc += partials[(int64_t)c * n + j];
  out[j] = acc;
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
  if (h % VW == 0 && h / VW <= 512 * kVPT) {
    ln_fwd_k<T, VW><<<(unsigned)rows, row_threads(h / VW), 0, st>>>(x, gain, bias, y, mean, rstd,
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
  const bool vec = h % VW == 0 && h / VW <= 512 * kVPT;
  require(vec || h <= 512 * kVPT, "bias_dropout_residual: hidden too large");
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
    int nt = (int)std::min<int64_t>(512, ((nvec + 31) / 32) * 32);
    ln_bwd_dx_k<T, VW><<<(unsigned)rows, nt, 0, st>>>(dy, x, mean, rstd, gain, resid_grad, dx,
                                                      (int)h);
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
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)num_chunks(rows, chunk_rows));
  colsum_partial_k<T><<<grid, 128, 0, st>>>(x, rows, n, ld, partials, chunk_rows);
  SPL_CHECK_LAUNCH();
}

void reduce_partials(const float* partials, int nchunks, int64_t n, float* out, bool accumulate,
                     cudaStream_t st) {
  if (n == 0) return;
  reduce_partials_k<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(partials, nchunks, n, out,
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
