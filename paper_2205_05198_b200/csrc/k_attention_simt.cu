// Attention core, SIMT flash-style kernels (fp32 execution dtype, and any shape).
//
// Forward (block.cpp:381-417 + attention_over_values 138-153): per (head, batch, query row)
// one warp streams the keys 32 at a time: S = q·k·scale, causal -inf, online softmax, the
// softmax-dropout keep bit from the counter RNG at the GLOBAL {a,b,s,s} coordinate
// ((g_head*b + b_j)*s + i)*s + j (block.cpp:392-394), O += P·keep/(1-p)·V.
// Selective recompute stores only O and the row LSE; the no-recompute regime additionally
// materialises softmax_out / mask / dropout_out.
//
// Backward (attention_interior_backward, block.cpp:159-193) recomputes P and keep from
// Q, K, LSE and the RNG (or reads the stored interior), with rowdot_i = dO_i·O_i:
//   dV_j = sum_i P_ij keep_ij/(1-p) dO_i, dP_ij = (dO_i·V_j) keep_ij/(1-p),
//   dS_ij = P_ij (dP_ij - rowdot_i), dQ_i = scale sum_j dS_ij K_j, dK_j = scale sum_i dS_ij Q_i.
// Two kernels (query-parallel dQ, key-parallel dK/dV) keep it free of atomics.
#include <cfloat>

#include "kernels.hpp"

namespace spl::k {

template <typename T>
void attn_fwd_tc(const AttnArgs& a, cudaStream_t st);
template <typename T>
void attn_bwd_tc(const AttnArgs& a, const void* dout, void* dqkv, float* delta, cudaStream_t st);
template <typename T>
bool attn_tc_supported(const AttnArgs& a);

namespace {

constexpr int kMaxHD = 256;
constexpr int kDPL = kMaxHD / 32;  // head-dim values per lane
constexpr int kWarps = 4;

__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// row index decomposition: r = ((hl * b) + bj) * s + i
struct RowId {
  int64_t hl, bj, i;
};
__device__ __forceinline__ RowId row_id(int64_t r, int64_t s, int64_t b) {
  RowId id;
  id.i = r % s;
  const int64_t t = r / s;
  id.bj = t % b;
  id.hl = t / b;
  return id;
}

template <typename T>
__device__ __forceinline__ float dot_row(const float* __restrict__ qs, const T* __restrict__ kr,
                                         int hd) {
  float acc = 0.f;
  for (int d = 0; d < hd; ++d) acc = fmaf(qs[d], to_f(kr[d]), acc);
  return acc;
}

template <typename T, bool MAT>
__global__ void __launch_bounds__(kWarps * 32) attn_fwd_simt_k(AttnArgs a) {
  __shared__ float qsh[kWarps][kMaxHD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t nrows = a.lh * a.b * a.s;
  if (r >= nrows) return;
  const RowId id = row_id(r, a.s, a.b);
  const int hd = (int)a.hd;
  const T* qkv = static_cast<const T*>(a.qkv);
  const int64_t qrow = (id.i * a.b + id.bj) * a.ld;
  for (int d = lane; d < hd; d += 32) qsh[warp][d] = to_f(qkv[qrow + a.qoff + id.hl * hd + d]);
  __syncwarp();
  const int64_t ghead = a.head_offset + id.hl;
  const uint64_t mrow = (uint64_t)(((ghead * a.b + id.bj) * a.s + id.i) * a.s);
  const int64_t kend = a.causal ? id.i + 1 : a.s;
  float o[kDPL];
#pragma unroll
  for (int u = 0; u < kDPL; ++u) o[u] = 0.f;
  float m = -INFINITY, l = 0.f;
  if (MAT) {  // pass 1: exact row statistics
    for (int64_t j0 = 0; j0 < kend; j0 += 32) {
      const int64_t jj = j0 + lane;
      float sc = -INFINITY;
      if (jj < kend)
        sc = dot_row<T>(qsh[warp], qkv + (jj * a.b + id.bj) * a.ld + a.koff + id.hl * hd, hd) *
             a.scale;
      const float mn = fmaxf(m, wmax(sc));
      const float p = jj < kend ? __expf(sc - mn) : 0.f;
      l = l * __expf(m - mn) + wsum(p);
      m = mn;
    }
  }
  const float inv_l = MAT ? 1.f / l : 0.f;
  for (int64_t j0 = 0; j0 < kend; j0 += 32) {
    const int64_t jj = j0 + lane;
    float sc = -INFINITY;
    if (jj < kend)
      sc = dot_row<T>(qsh[warp], qkv + (jj * a.b + id.bj) * a.ld + a.koff + id.hl * hd, hd) *
           a.scale;
    const bool keep = jj < kend ? drop_keep(a.drop, mrow + (uint64_t)jj) : false;
    float pd;
    if (MAT) {
      const float p = jj < kend ? __expf(sc - m) * inv_l : 0.f;
      pd = keep ? p * a.drop.inv_keep : 0.f;
      const int64_t mi = ((id.hl * a.b + id.bj) * a.s + id.i) * a.s + jj;
      if (jj < a.s && jj >= kend) {  // causal zeros of the stored interior
        static_cast<T*>(a.sm)[mi] = from_f<T>(0.f);
        a.mask[mi] = drop_keep(a.drop, mrow + (uint64_t)jj) ? 1 : 0;
        static_cast<T*>(a.sd)[mi] = from_f<T>(0.f);
      } else if (jj < kend) {
        static_cast<T*>(a.sm)[mi] = from_f<T>(p);
        a.mask[mi] = keep ? 1 : 0;
        static_cast<T*>(a.sd)[mi] = from_f<T>(pd);
      }
    } else {
      const float mn = fmaxf(m, wmax(sc));
      const float p = jj < kend ? __expf(sc - mn) : 0.f;
      const float corr = __expf(m - mn);
      l = l * corr + wsum(p);
      m = mn;
#pragma unroll
      for (int u = 0; u < kDPL; ++u) o[u] *= corr;
      pd = keep ? p * a.drop.inv_keep : 0.f;
    }
    const int nk = (int)(kend - j0 < 32 ? kend - j0 : 32);
    for (int kk = 0; kk < nk; ++kk) {
      const float pk = __shfl_sync(0xffffffffu, pd, kk);
      const T* vr = qkv + ((j0 + kk) * a.b + id.bj) * a.ld + a.voff + id.hl * hd;
#pragma unroll
      for (int u = 0; u < kDPL; ++u) {
        const int d = lane + 32 * u;
        if (d < hd) o[u] = fmaf(pk, to_f(vr[d]), o[u]);
      }
    }
  }
  if (MAT && a.causal) {  // remaining (j >= kend) blocks of the stored interior
    for (int64_t jj = ((kend + 31) / 32) * 32 + lane; jj < a.s; jj += 32) {
      const int64_t mi = ((id.hl * a.b + id.bj) * a.s + id.i) * a.s + jj;
      static_cast<T*>(a.sm)[mi] = from_f<T>(0.f);
      a.mask[mi] = drop_keep(a.drop, mrow + (uint64_t)jj) ? 1 : 0;
      static_cast<T*>(a.sd)[mi] = from_f<T>(0.f);
    }
  }
  const float fin = MAT ? 1.f : 1.f / l;
  T* orow = static_cast<T*>(a.o) + (id.i * a.b + id.bj) * a.ldo + id.hl * hd;
#pragma unroll
  for (int u = 0; u < kDPL; ++u) {
    const int d = lane + 32 * u;
    if (d < hd) orow[d] = from_f<T>(o[u] * fin);
  }
  if (lane == 0 && a.lse) a.lse[r] = m + logf(l);
}

// delta_r = dO_r · O_r
template <typename T>
__global__ void attn_delta_k(AttnArgs a, const T* __restrict__ dout, float* __restrict__ delta) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kWarps + warp;
  if (r >= a.lh * a.b * a.s) return;
  const RowId id = row_id(r, a.s, a.b);
  const int64_t off = (id.i * a.b + id.bj) * a.ldo + id.hl * a.hd;
  const T* o = static_cast<const T*>(a.o);
  float acc = 0.f;
  for (int d = lane; d < a.hd; d += 32) acc += to_f(dout[off + d]) * to_f(o[off + d]);
  acc = wsum(acc);
  if (lane == 0) delta[r] = acc;
}

// P, keep for (query row of id, key jj); stored or recomputed.
template <typename T, bool STORED>
__device__ __forceinline__ void p_keep(const AttnArgs& a, const RowId& id, int64_t jj,
                                       const float* qs, float lse, uint64_t mrow, float& p,
                                       bool& keep) {
  if (STORED) {
    const int64_t mi = ((id.hl * a.b + id.bj) * a.s + id.i) * a.s + jj;
    p = to_f(static_cast<const T*>(a.sm)[mi]);
    keep = a.mask[mi] != 0;
  } else {
    const T* qkv = static_cast<const T*>(a.qkv);
    const float sc =
        dot_row<T>(qs, qkv + (jj * a.b + id.bj) * a.ld + a.koff + id.hl * a.hd, (int)a.hd) *
        a.scale;
    p = __expf(sc - lse);
    keep = drop_keep(a.drop, mrow + (uint64_t)jj);
  }
}

template <typename T, bool STORED>
__global__ void __launch_bounds__(kWarps * 32) attn_bwd_dq_k(AttnArgs a, const T* __restrict__ dout,
                                                            T* __restrict__ dqkv,
                                                            const float* __restrict__ delta) {
  __shared__ float qsh[kWarps][kMaxHD];
  __shared__ float dosh[kWarps][kMaxHD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kWarps + warp;
  if (r >= a.lh * a.b * a.s) return;
  const RowId id = row_id(r, a.s, a.b);
  const int hd = (int)a.hd;
  const T* qkv = static_cast<const T*>(a.qkv);
  const int64_t row = id.i * a.b + id.bj;
  for (int d = lane; d < hd; d += 32) {
    qsh[warp][d] = to_f(qkv[row * a.ld + a.qoff + id.hl * hd + d]);
    dosh[warp][d] = to_f(dout[row * a.ldo + id.hl * hd + d]);
  }
  __syncwarp();
  const float lse = a.lse ? a.lse[r] : 0.f, dlt = delta[r];
  const uint64_t mrow =
      (uint64_t)((((a.head_offset + id.hl) * a.b + id.bj) * a.s + id.i) * a.s);
  const int64_t kend = a.causal ? id.i + 1 : a.s;
  float dq[kDPL];
#pragma unroll
  for (int u = 0; u < kDPL; ++u) dq[u] = 0.f;
  for (int64_t j0 = 0; j0 < kend; j0 += 32) {
    const int64_t jj = j0 + lane;
    float ds = 0.f;
    if (jj < kend) {
      float p;
      bool keep;
      p_keep<T, STORED>(a, id, jj, qsh[warp], lse, mrow, p, keep);
      const float dpd =
          dot_row<T>(dosh[warp], qkv + (jj * a.b + id.bj) * a.ld + a.voff + id.hl * hd, hd);
      const float dp = keep ? dpd * a.drop.inv_keep : 0.f;
      ds = p * (dp - dlt);
    }
    const int nk = (int)(kend - j0 < 32 ? kend - j0 : 32);
    for (int kk = 0; kk < nk; ++kk) {
      const float dsk = __shfl_sync(0xffffffffu, ds, kk);
      const T* kr = qkv + ((j0 + kk) * a.b + id.bj) * a.ld + a.koff + id.hl * hd;
#pragma unroll
      for (int u = 0; u < kDPL; ++u) {
        const int d = lane + 32 * u;
        if (d < hd) dq[u] = fmaf(dsk, to_f(kr[d]), dq[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kDPL; ++u) {
    const int d = lane + 32 * u;
    if (d < hd) dqkv[row * a.ld + a.qoff + id.hl * hd + d] = from_f<T>(dq[u] * a.scale);
  }
}

template <typename T, bool STORED>
__global__ void __launch_bounds__(kWarps * 32) attn_bwd_dkdv_k(AttnArgs a,
                                                              const T* __restrict__ dout,
                                                              T* __restrict__ dqkv,
                                                              const float* __restrict__ delta) {
  __shared__ float ksh[kWarps][kMaxHD];
  __shared__ float vsh[kWarps][kMaxHD];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kWarps + warp;  // key row id: ((hl*b)+bj)*s + jj
  if (r >= a.lh * a.b * a.s) return;
  const RowId kid = row_id(r, a.s, a.b);
  const int64_t jj = kid.i;
  const int hd = (int)a.hd;
  const T* qkv = static_cast<const T*>(a.qkv);
  const int64_t krow = jj * a.b + kid.bj;
  for (int d = lane; d < hd; d += 32) {
    ksh[warp][d] = to_f(qkv[krow * a.ld + a.koff + kid.hl * hd + d]);
    vsh[warp][d] = to_f(qkv[krow * a.ld + a.voff + kid.hl * hd + d]);
  }
  __syncwarp();
  float dk[kDPL], dv[kDPL];
#pragma unroll
  for (int u = 0; u < kDPL; ++u) dk[u] = dv[u] = 0.f;
  const int64_t istart = a.causal ? jj : 0;
  for (int64_t i0 = istart; i0 < a.s; i0 += 32) {
    const int64_t ii = i0 + lane;
    float ds = 0.f, pd = 0.f;
    if (ii < a.s) {
      RowId qid{kid.hl, kid.bj, ii};
      const int64_t qr = (kid.hl * a.b + kid.bj) * a.s + ii;
      const uint64_t mrow =
          (uint64_t)((((a.head_offset + kid.hl) * a.b + kid.bj) * a.s + ii) * a.s);
      float p;
      bool keep;
      if (STORED) {
        const int64_t mi = qr * a.s + jj;
        p = to_f(static_cast<const T*>(a.sm)[mi]);
        keep = a.mask[mi] != 0;
      } else {
        const float sc =
            dot_row<T>(ksh[warp], qkv + (ii * a.b + kid.bj) * a.ld + a.qoff + kid.hl * hd, hd) *
            a.scale;
        p = __expf(sc - a.lse[qr]);
        keep = drop_keep(a.drop, mrow + (uint64_t)jj);
      }
      (void)qid;
      const float dpd =
          dot_row<T>(vsh[warp], dout + (ii * a.b + kid.bj) * a.ldo + kid.hl * hd, hd);
      const float dp = keep ? dpd * a.drop.inv_keep : 0.f;
      ds = p * (dp - delta[qr]);
      pd = keep ? p * a.drop.inv_keep : 0.f;
    }
    const int ni = (int)(a.s - i0 < 32 ? a.s - i0 : 32);
    for (int q = 0; q < ni; ++q) {
      const float dsq = __shfl_sync(0xffffffffu, ds, q);
      const float pdq = __shfl_sync(0xffffffffu, pd, q);
      const int64_t row = (i0 + q) * a.b + kid.bj;
      const T* qr_ = qkv + row * a.ld + a.qoff + kid.hl * hd;
      const T* dr = dout + row * a.ldo + kid.hl * hd;
#pragma unroll
      for (int u = 0; u < kDPL; ++u) {
        const int d = lane + 32 * u;
        if (d < hd) {
          dk[u] = fmaf(dsq, to_f(qr_[d]), dk[u]);
          dv[u] = fmaf(pdq, to_f(dr[d]), dv[u]);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kDPL; ++u) {
    const int d = lane + 32 * u;
    if (d < hd) {
      dqkv[krow * a.ld + a.koff + kid.hl * hd + d] = from_f<T>(dk[u] * a.scale);
      dqkv[krow * a.ld + a.voff + kid.hl * hd + d] = from_f<T>(dv[u]);
    }
  }
}

}  // namespace

template <typename T>
void attn_fwd(const AttnArgs& a, cudaStream_t st) {
  require(a.hd <= kMaxHD, "attention: head_dim > 256 unsupported");
  if (attn_tc_supported<T>(a)) {
    attn_fwd_tc<T>(a, st);
    return;
  }
  const int64_t rows = a.lh * a.b * a.s;
  const unsigned grid = (unsigned)((rows + kWarps - 1) / kWarps);
  if (a.sm) attn_fwd_simt_k<T, true><<<grid, kWarps * 32, 0, st>>>(a);
  else attn_fwd_simt_k<T, false><<<grid, kWarps * 32, 0, st>>>(a);
  SPL_CHECK_LAUNCH();
}

template <typename T>
void attn_bwd(const AttnArgs& a, const void* dout, void* dqkv, float* delta, cudaStream_t st) {
  require(a.hd <= kMaxHD, "attention: head_dim > 256 unsupported");
  if (attn_tc_supported<T>(a)) {
    attn_bwd_tc<T>(a, dout, dqkv, delta, st);
    return;
  }
  const int64_t rows = a.lh * a.b * a.s;
  const unsigned grid = (unsigned)((rows + kWarps - 1) / kWarps);
  const T* d = static_cast<const T*>(dout);
  T* g = static_cast<T*>(dqkv);
  attn_delta_k<T><<<grid, kWarps * 32, 0, st>>>(a, d, delta);
  if (a.sm) {
    attn_bwd_dq_k<T, true><<<grid, kWarps * 32, 0, st>>>(a, d, g, delta);
    attn_bwd_dkdv_k<T, true><<<grid, kWarps * 32, 0, st>>>(a, d, g, delta);
  } else {
    attn_bwd_dq_k<T, false><<<grid, kWarps * 32, 0, st>>>(a, d, g, delta);
    attn_bwd_dkdv_k<T, false><<<grid, kWarps * 32, 0, st>>>(a, d, g, delta);
  }
  SPL_CHECK_LAUNCH();
}

template void attn_fwd<float>(const AttnArgs&, cudaStream_t);
template void attn_fwd<bf16>(const AttnArgs&, cudaStream_t);
template void attn_bwd<float>(const AttnArgs&, const void*, void*, float*, cudaStream_t);
template void attn_bwd<bf16>(const AttnArgs&, const void*, void*, float*, cudaStream_t);

// Tensor-core kernels are provided for bf16 only (k_attention_tc.cu).
template <>
bool attn_tc_supported<float>(const AttnArgs&) {
  return false;
}
template <>
void attn_fwd_tc<float>(const AttnArgs&, cudaStream_t) {}
template <>
void attn_bwd_tc<float>(const AttnArgs&, const void*, void*, float*, cudaStream_t) {}

}  // namespace spl::k
