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
#include <type_traits>

#include "kernels.hpp"

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

// =====================================================================================
// forward
// =====================================================================================
template <int HD>
__global__ void __launch_bounds__(128) fa_fwd(AttnArgs a) {
  constexpr int BM = 64, BN = 64, LDS = HD + 8, NT = 128;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  bf16* Qs = reinterpret_cast<bf16*>(smem_raw);
  bf16* Ks = Qs + BM * LDS;           // [2][BN][LDS]
  bf16* Vs = Ks + 2 * BN * LDS;       // [2][BN][LDS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int64_t q0 = (int64_t)blockIdx.x * BM;
  const int64_t hl = blockIdx.y / a.b, bj = blockIdx.y % a.b;
  const bf16* qkv = static_cast<const bf16*>(a.qkv);
  const bf16* base = qkv + bj * a.ld;  // row i of this batch at base + i*b*ld
  const int64_t rstride = a.b * a.ld;
  const int64_t qcol = a.qoff + hl * HD, kcol = a.koff + hl * HD, vcol = a.voff + hl * HD;

  const int64_t kv_end = a.causal ? (a.s < q0 + BM ? a.s : q0 + BM) : a.s;
  const int nkv = (int)((kv_end + BN - 1) / BN);

  load_tile<HD, BM, NT>(Qs, base, q0, a.s, rstride, qcol);
  load_tile<HD, BN, NT>(Ks, base, 0, a.s, rstride, kcol);
  load_tile<HD, BN, NT>(Vs, base, 0, a.s, rstride, vcol);
  cp_commit();

  uint32_t qf[HD / 16][4];
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  const float sl2 = a.scale * kLog2e;
  const int64_t row0 = q0 + warp * 16 + g;  // this thread's rows: row0, row0 + 8
  const int64_t ghead = a.head_offset + hl;
  const uint64_t mbase = (uint64_t)((ghead * a.b + bj) * a.s);
  const uint64_t mrow0 = (mbase + (uint64_t)row0) * (uint64_t)a.s;
  const uint64_t mrow1 = (mbase + (uint64_t)row0 + 8) * (uint64_t)a.s;

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
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(qf[kk], Qs + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
    }
    const bf16* Kb = Ks + buf * BN * LDS;
    const bf16* Vb = Vs + buf * BN * LDS;
    float sacc[BN / 8][4];
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
    // scale, bounds/causal mask, online softmax (log2 domain)
    const int64_t k0 = (int64_t)jb * BN;
    float mx[2] = {m[0], m[1]};
#pragma unroll
    for (int nb = 0; nb < BN / 8; ++nb) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t key = k0 + nb * 8 + 2 * tq + (e & 1);
        const int64_t qr = row0 + (e >> 1) * 8;
        float v = sacc[nb][e] * sl2;
        if (key >= a.s || (a.causal && key > qr)) v = -INFINITY;
        sacc[nb][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float mnew = mx[r];
      corr[r] = (m[r] == -INFINITY) ? 0.f : exp2f(m[r] - mnew);
      m[r] = mnew;
      l[r] *= corr[r];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= corr[0]; o[i][1] *= corr[0];
      o[i][2] *= corr[1]; o[i][3] *= corr[1];
    }
    uint32_t pa[BN / 16][4];
#pragma unroll
    for (int nb = 0; nb < BN / 8; ++nb) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const float mr = m[r] == -INFINITY ? 0.f : m[r];
        const float pv = exp2f(sacc[nb][e] - mr);
        l[r] += pv;
        const int64_t key = k0 + nb * 8 + 2 * tq + (e & 1);
        bool keep = false;
        if (pv != 0.f) keep = drop_keep(a.drop, (r ? mrow1 : mrow0) + (uint64_t)key);
        p[e] = keep ? pv * a.drop.inv_keep : 0.f;
      }
      const int kk2 = nb >> 1, hi = nb & 1;
      pa[kk2][hi * 2 + 0] = pack_bf16(p[0], p[1]);
      pa[kk2][hi * 2 + 1] = pack_bf16(p[2], p[3]);
    }
    // O += P̃ · V
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
  // finalize
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
  }
  bf16* out = static_cast<bf16*>(a.o);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int64_t qr = row0 + r * 8;
    if (qr >= a.s) continue;
    const float inv = 1.f / l[r];
    bf16* orow = out + (qr * a.b + bj) * a.ldo + hl * HD;
#pragma unroll
    for (int db = 0; db < HD / 8; ++db) {
      const uint32_t v = pack_bf16(o[db][2 * r] * inv, o[db][2 * r + 1] * inv);
      *reinterpret_cast<uint32_t*>(orow + db * 8 + 2 * tq) = v;
    }
    if (tq == 0 && a.lse) a.lse[(hl * a.b + bj) * a.s + qr] = (m[r] + log2f(l[r])) * kLn2;
  }
}

// =====================================================================================
// backward: delta = rowsum(dO ∘ O)
// =====================================================================================
template <int HD>
__global__ void fa_delta(AttnArgs a, const bf16* __restrict__ dout, float* __restrict__ delta) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 4 + warp;  // ((hl*b)+bj)*s + i
  if (r >= a.lh * a.b * a.s) return;
  const int64_t i = r % a.s, t = r / a.s, bj = t % a.b, hl = t / a.b;
  const int64_t off = (i * a.b + bj) * a.ldo + hl * HD;
  const bf16* o = static_cast<const bf16*>(a.o);
  float acc = 0.f;
  for (int d = lane * 2; d < HD; d += 64) {
    const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(dout + off + d);
    const __nv_bfloat162 y = *reinterpret_cast<const __nv_bfloat162*>(o + off + d);
    acc += __bfloat162float(x.x) * __bfloat162float(y.x) + __bfloat162float(x.y) * __bfloat162float(y.y);
  }
#pragma unroll
  for (int k = 16; k; k >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, k);
  if (lane == 0) delta[r] = acc;
}

// =====================================================================================
// backward: dK, dV (key-parallel)
// =====================================================================================
template <int HD>
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
  const int64_t k0 = (int64_t)blockIdx.x * BK_;
  const int64_t hl = blockIdx.y / a.b, bj = blockIdx.y % a.b;
  const bf16* qkv = static_cast<const bf16*>(a.qkv);
  const bf16* base = qkv + bj * a.ld;
  const bf16* dbase = dout + bj * a.ldo;
  const int64_t rstride = a.b * a.ld, dstride = a.b * a.ldo;
  const int64_t qcol = a.qoff + hl * HD, kcol = a.koff + hl * HD, vcol = a.voff + hl * HD;
  const int64_t rowbase = (hl * a.b + bj) * a.s;  // lse/delta row index base
  const float sl2 = a.scale * kLog2e;
  const uint64_t mbase = (uint64_t)(((a.head_offset + hl) * a.b + bj) * a.s);

  const int64_t q_start = a.causal ? (k0 / BQ) * BQ : 0;
  const int nq = (int)((a.s - q_start + BQ - 1) / BQ);

  auto load_q = [&](int it, int buf) {
    const int64_t qb = q_start + (int64_t)it * BQ;
    load_tile<HD, BQ, NT>(Qs + buf * BQ * LDS, base, qb, a.s, rstride, qcol);
    load_tile<HD, BQ, NT>(Ds + buf * BQ * LDS, dbase, qb, a.s, dstride, hl * HD);
    if (threadIdx.x < BQ) {
      const int64_t q = qb + threadIdx.x;
      lse_s[buf * BQ + threadIdx.x] = q < a.s ? a.lse[rowbase + q] : INFINITY;
      dl_s[buf * BQ + threadIdx.x] = q < a.s ? delta[rowbase + q] : 0.f;
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
  const int64_t key0 = k0 + warp * 16 + g;  // rows of this thread: key0, key0 + 8

  for (int it = 0; it < nq; ++it) {
    const int buf = it & 1;
    __syncthreads();  // previous iteration done with buf^1 (and lse/delta slots)
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
    const int64_t qb = q_start + (int64_t)it * BQ;
    // Sᵀ = K Qᵀ and dPᵀ = V dOᵀ : [16 keys × 32 queries] per warp
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
    // Pᵀ, keepᵀ, dSᵀ
    uint32_t pa[BQ / 16][4], da[BQ / 16][4];
#pragma unroll
    for (int nb = 0; nb < BQ / 8; ++nb) {
      float pd[4], ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = nb * 8 + 2 * tq + (e & 1);
        const int64_t q = qb + qi;
        const int64_t key = key0 + (e >> 1) * 8;
        float p = 0.f;
        bool keep = false;
        if (q < a.s && key < a.s && !(a.causal && key > q)) {
          p = exp2f(st[nb][e] * sl2 - lq[qi] * kLog2e);
          if (p != 0.f) keep = drop_keep(a.drop, (mbase + (uint64_t)q) * (uint64_t)a.s + (uint64_t)key);
        }
        pd[e] = keep ? p * a.drop.inv_keep : 0.f;
        const float dp = keep ? dpt[nb][e] * a.drop.inv_keep : 0.f;
        ds[e] = p * (dp - dq_[qi]);
      }
      const int kk2 = nb >> 1, hi = nb & 1;
      pa[kk2][hi * 2 + 0] = pack_bf16(pd[0], pd[1]);
      pa[kk2][hi * 2 + 1] = pack_bf16(pd[2], pd[3]);
      da[kk2][hi * 2 + 0] = pack_bf16(ds[0], ds[1]);
      da[kk2][hi * 2 + 1] = pack_bf16(ds[2], ds[3]);
    }
    // dV += P̃ᵀ dO ; dK += dSᵀ Q
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
    const int64_t key = key0 + r * 8;
    if (key >= a.s) continue;
    bf16* row = dqkv + (key * a.b + bj) * a.ld;
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
// backward: dQ (query-parallel)
// =====================================================================================
template <int HD>
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
  const int64_t q0 = (int64_t)blockIdx.x * BM;
  const int64_t hl = blockIdx.y / a.b, bj = blockIdx.y % a.b;
  const bf16* qkv = static_cast<const bf16*>(a.qkv);
  const bf16* base = qkv + bj * a.ld;
  const bf16* dbase = dout + bj * a.ldo;
  const int64_t rstride = a.b * a.ld, dstride = a.b * a.ldo;
  const int64_t qcol = a.qoff + hl * HD, kcol = a.koff + hl * HD, vcol = a.voff + hl * HD;
  const int64_t rowbase = (hl * a.b + bj) * a.s;
  const float sl2 = a.scale * kLog2e;
  const uint64_t mbase = (uint64_t)(((a.head_offset + hl) * a.b + bj) * a.s);
  const int64_t kv_end = a.causal ? (a.s < q0 + BM ? a.s : q0 + BM) : a.s;
  const int nkv = (int)((kv_end + BN - 1) / BN);

  load_tile<HD, BM, NT>(Qs, base, q0, a.s, rstride, qcol);
  load_tile<HD, BM, NT>(Ds, dbase, q0, a.s, dstride, hl * HD);
  load_tile<HD, BN, NT>(Ks, base, 0, a.s, rstride, kcol);
  load_tile<HD, BN, NT>(Vs, base, 0, a.s, rstride, vcol);
  cp_commit();

  const int64_t row0 = q0 + warp * 16 + g;
  float lse[2], dl[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int64_t q = row0 + r * 8;
    lse[r] = q < a.s ? a.lse[rowbase + q] * kLog2e : INFINITY;
    dl[r] = q < a.s ? delta[rowbase + q] : 0.f;
  }
  const uint64_t mrow[2] = {(mbase + (uint64_t)row0) * (uint64_t)a.s,
                            (mbase + (uint64_t)row0 + 8) * (uint64_t)a.s};
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
    const int64_t kb0 = (int64_t)jb * BN;
    uint32_t da[BN / 16][4];
#pragma unroll
    for (int nb = 0; nb < BN / 8; ++nb) {
      float ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const int64_t key = kb0 + nb * 8 + 2 * tq + (e & 1);
        const int64_t q = row0 + r * 8;
        float p = 0.f;
        bool keep = false;
        if (q < a.s && key < a.s && !(a.causal && key > q)) {
          p = exp2f(sc[nb][e] * sl2 - lse[r]);
          if (p != 0.f) keep = drop_keep(a.drop, mrow[r] + (uint64_t)key);
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
    const int64_t q = row0 + r * 8;
    if (q >= a.s) continue;
    bf16* row = dqkv + (q * a.b + bj) * a.ld + qcol;
#pragma unroll
    for (int db = 0; db < HD / 8; ++db)
      *reinterpret_cast<uint32_t*>(row + db * 8 + 2 * tq) =
          pack_bf16(dq[db][2 * r] * a.scale, dq[db][2 * r + 1] * a.scale);
  }
}

template <int HD>
void launch_fwd(const AttnArgs& a, cudaStream_t st) {
  constexpr int LDS = HD + 8;
  const int smem = (64 * LDS + 4 * 64 * LDS) * 2;
  static bool once = [&] {
    SPL_CUDA(cudaFuncSetAttribute(fa_fwd<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return true;
  }();
  (void)once;
  dim3 grid((unsigned)((a.s + 63) / 64), (unsigned)(a.lh * a.b));
  fa_fwd<HD><<<grid, 128, smem, st>>>(a);
  SPL_CHECK_LAUNCH();
}

template <int HD>
void launch_bwd(const AttnArgs& a, const bf16* dout, bf16* dqkv, float* delta, cudaStream_t st) {
  constexpr int LDS = HD + 8;
  const int64_t rows = a.lh * a.b * a.s;
  fa_delta<HD><<<(unsigned)((rows + 3) / 4), 128, 0, st>>>(a, dout, delta);
  SPL_CHECK_LAUNCH();
  const int smem_kv = (2 * 64 * LDS + 4 * 32 * LDS) * 2 + 4 * 32 * 4;
  const int smem_q = (2 * 64 * LDS + 4 * 32 * LDS) * 2;
  static bool once = [&] {
    SPL_CUDA(cudaFuncSetAttribute(fa_bwd_dkdv<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv));
    SPL_CUDA(cudaFuncSetAttribute(fa_bwd_dq<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q));
    return true;
  }();
  (void)once;
  dim3 grid((unsigned)((a.s + 63) / 64), (unsigned)(a.lh * a.b));
  fa_bwd_dkdv<HD><<<grid, 128, smem_kv, st>>>(a, dout, dqkv, delta);
  SPL_CHECK_LAUNCH();
  fa_bwd_dq<HD><<<grid, 128, smem_q, st>>>(a, dout, dqkv, delta);
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
  return hd_ok && a.ld % 8 == 0 && a.ldo % 8 == 0 && a.qoff % 8 == 0 && a.koff % 8 == 0 &&
         a.voff % 8 == 0 && aligned16(a.qkv) && aligned16(a.o) && a.lse != nullptr;
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
  SPL_HD_SWITCH(a.hd, launch_fwd<HD>(a, st));
}

template <>
void attn_bwd_tc<bf16>(const AttnArgs& a, const void* dout, void* dqkv, float* delta,
                       cudaStream_t st) {
  SPL_HD_SWITCH(a.hd, launch_bwd<HD>(a, static_cast<const bf16*>(dout), static_cast<bf16*>(dqkv),
                                     delta, st));
}

}  // namespace spl::k
