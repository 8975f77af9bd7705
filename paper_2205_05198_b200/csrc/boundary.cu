// Free-standing entry points of the reference seqpar API that are not a layer call:
//   attention_interior(q, k, cfg, head_offset, local_heads)   block.hpp:100-101, block.cpp:381-417
//   all_gather / reduce_scatter / all_reduce over rank shards  collectives.hpp:57-62,
//                                                             collectives.cpp:21-73
// on device buffers (include/spl.h). The collectives run the reference's simulated-rank group on
// one GPU: gathers are strided copies, reductions sum the partials in rank order 0..t-1 (the
// determinism contract of collectives.hpp:54-56) — in fp64 that is bit-identical to the
// reference's ordered_sum, in fp32/bf16 it is one fp32 accumulation rounded once.
#include <cstring>
#include <string>

#include "../../include/spl.h"
#include "common.hpp"
#include "kernels.hpp"
#include "rng.cuh"

namespace spl {
namespace {

constexpr int kMaxRanks = 64;

struct RankPtrs {
  const void* p[kMaxRanks];
};

struct AxisBlocks {  // tensor.cpp:150-166
  int64_t outer = 1, axis = 1, inner = 1;
};

AxisBlocks axis_blocks(const int64_t* shape, int ndim, int axis) {
  if (axis < 0 || axis >= ndim) raise(SPL_EINVAL, "axis out of range");
  AxisBlocks b;
  for (int i = 0; i < ndim; ++i) {
    if (shape[i] < 0) raise(SPL_EINVAL, "negative tensor dimension");
    if (i < axis) b.outer *= shape[i];
    else if (i == axis) b.axis = shape[i];
    else b.inner *= shape[i];
  }
  return b;
}

size_t esize(int dtype) {
  switch (dtype) {
    case SPL_DTYPE_F32: return 4;
    case SPL_DTYPE_BF16: return 2;
    case SPL_DTYPE_F64: return 8;
  }
  raise(SPL_EINVAL, "unknown dtype");
}

template <typename T, typename Acc>
__device__ __forceinline__ Acc load_as(const T* p, int64_t i) {
  if constexpr (std::is_same_v<T, bf16>) return (Acc)__bfloat162float(p[i]);
  else return (Acc)p[i];
}
template <typename T, typename Acc>
__device__ __forceinline__ T store_as(Acc v) {
  if constexpr (std::is_same_v<T, bf16>) return __float2bfloat16_rn((float)v);
  else return (T)v;
}

// out[o, r*piece_out + a, i] (or the whole tensor when scatter == 0) = Σ_{q=0..t-1} in_q[...]
// summed in rank order. Element e of rank r's output piece: (o, a, i) over {outer, piece, inner}.
template <typename T, typename Acc>
__global__ void __launch_bounds__(256) ordered_sum_k(RankPtrs in, int t, void* out, int64_t n,
                                                     int64_t piece, int64_t inner, int64_t full_axis,
                                                     int64_t piece_offset) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    const int64_t i = e % inner;
    const int64_t oa = e / inner;
    const int64_t a = oa % piece;
    const int64_t o = oa / piece;
    const int64_t src = (o * full_axis + piece_offset + a) * inner + i;
    Acc acc = load_as<T, Acc>(static_cast<const T*>(in.p[0]), src);
    for (int q = 1; q < t; ++q) acc += load_as<T, Acc>(static_cast<const T*>(in.p[q]), src);
    static_cast<T*>(out)[e] = store_as<T, Acc>(acc);
  }
}

template <typename T, typename Acc>
void launch_sum(const RankPtrs& in, int t, void* out, int64_t n, int64_t piece, int64_t inner,
                int64_t full_axis, int64_t off, cudaStream_t st) {
  if (n == 0) return;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 16);
  ordered_sum_k<T, Acc><<<(unsigned)blocks, 256, 0, st>>>(in, t, out, n, piece, inner, full_axis, off);
  SPL_CHECK_LAUNCH();
}

void sum_dispatch(int dtype, const RankPtrs& in, int t, void* out, int64_t n, int64_t piece,
                  int64_t inner, int64_t full_axis, int64_t off, cudaStream_t st) {
  switch (dtype) {
    case SPL_DTYPE_F64: launch_sum<double, double>(in, t, out, n, piece, inner, full_axis, off, st); break;
    case SPL_DTYPE_F32: launch_sum<float, float>(in, t, out, n, piece, inner, full_axis, off, st); break;
    case SPL_DTYPE_BF16: launch_sum<bf16, float>(in, t, out, n, piece, inner, full_axis, off, st); break;
    default: raise(SPL_EINVAL, "unknown dtype");
  }
}

RankPtrs rank_ptrs(const void* const* shards, int t, const char* op) {
  if (t < 1 || shards == nullptr) raise(SPL_EINVAL, std::string(op) + ": empty rank group");
  if (t > kMaxRanks) raise(SPL_EINVAL, std::string(op) + ": more than 64 ranks");
  RankPtrs p{};
  for (int r = 0; r < t; ++r) {
    if (shards[r] == nullptr) raise(SPL_EINVAL, std::string(op) + ": null shard");
    p.p[r] = shards[r];
  }
  return p;
}

// CommLog ring-element model (collectives.cpp:30-38): steps × (logical / ranks) × (ranks − 1).
void log_ring(int64_t* log, int tag, int field, int64_t logical, int64_t t, int64_t steps) {
  if (log == nullptr) return;
  if (tag < 0 || tag > 2) raise(SPL_EINVAL, "unknown comm tag");
  log[4 * tag + field] += 1;
  log[4 * tag + 3] += steps * (logical / t) * (t - 1);
}

struct Scope {
  int prev = 0;
  explicit Scope(int dev) {
    SPL_CUDA(cudaGetDevice(&prev));
    SPL_CUDA(cudaSetDevice(dev));
  }
  ~Scope() { cudaSetDevice(prev); }
};

template <typename T>
void interior_impl(const spl_layer_desc& d, const void* q, const void* k, int64_t head_offset,
                   int64_t lh, void* sm, uint8_t* mask, void* sd, cudaStream_t st) {
  const int64_t s = d.seq, b = d.batch, hd = d.hidden / d.heads, lw = lh * hd;
  const int64_t rows = s * b;
  T* qkv = nullptr;
  T* o = nullptr;
  uint32_t* bits = nullptr;
  const int64_t words = k::keepbits_words(lh, b, s);
  SPL_CUDA(cudaMallocAsync(&qkv, sizeof(T) * rows * 3 * lw, st));
  SPL_CUDA(cudaMallocAsync(&o, sizeof(T) * rows * lw, st));
  SPL_CUDA(cudaMallocAsync(&bits, sizeof(uint32_t) * std::max<int64_t>(words, 1), st));
  // pack [Q | K | 0] rows of the fused layout the attention kernels read
  SPL_CUDA(cudaMemsetAsync(qkv, 0, sizeof(T) * rows * 3 * lw, st));
  SPL_CUDA(cudaMemcpy2DAsync(qkv, sizeof(T) * 3 * lw, q, sizeof(T) * lw, sizeof(T) * lw, rows,
                             cudaMemcpyDeviceToDevice, st));
  SPL_CUDA(cudaMemcpy2DAsync(qkv + lw, sizeof(T) * 3 * lw, k, sizeof(T) * lw, sizeof(T) * lw, rows,
                             cudaMemcpyDeviceToDevice, st));
  k::AttnArgs a;
  a.s = s; a.b = b; a.lh = lh; a.hd = hd;
  a.head_offset = head_offset;
  a.heads_total = d.heads;
  a.qkv = qkv; a.ld = 3 * lw; a.qoff = 0; a.koff = lw; a.voff = 2 * lw;
  a.o = o; a.ldo = lw;
  a.scale = (float)(1.0 / std::sqrt((double)hd));
  a.causal = d.causal;
  a.drop = make_drop_key(d.seed, d.layer_index, kSoftmaxDrop, d.microbatch, d.dropout_p);
  a.lse = nullptr;
  a.sm = sm; a.mask = mask; a.sd = sd;
  a.keepbits = bits;
  k::attn_keep_bits(a, st);
  k::attn_fwd<T>(a, st);
  SPL_CUDA(cudaFreeAsync(qkv, st));
  SPL_CUDA(cudaFreeAsync(o, st));
  SPL_CUDA(cudaFreeAsync(bits, st));
}

}  // namespace
}  // namespace spl

namespace {
template <typename F>
int bguard(F&& f) {
  return spl::c_guard(std::forward<F>(f));
}
}  // namespace

extern "C" {

int spl_attention_interior_qk(const spl_layer_desc* d, int device, const void* q, const void* k,
                              int64_t head_offset, int64_t local_heads, void* softmax_out,
                              uint8_t* dropout_mask, void* dropout_out, void* stream) {
  return bguard([&] {
    using namespace spl;
    require(d != nullptr, "null desc");
    require(q && k && softmax_out && dropout_mask && dropout_out, "null buffer");
    require(d->heads > 0 && d->hidden % d->heads == 0, "hidden not divisible by heads");
    require(d->seq > 0 && d->batch > 0, "seq and batch must be positive");
    // mask_slice(…, parts = heads/local_heads, index = head_offset/local_heads) (block.cpp:392-394)
    require(local_heads >= 1 && d->heads % local_heads == 0, "mask axis not divisible");
    require(head_offset >= 0 && head_offset % local_heads == 0 && head_offset < d->heads,
            "slice index out of range");
    require(d->dropout_p >= 0.0 && d->dropout_p < 1.0, "dropout probability must lie in [0, 1)");
    require(d->dtype == SPL_DTYPE_F32 || d->dtype == SPL_DTYPE_BF16, "dtype must be f32 or bf16");
    Scope sc(device);
    auto st = static_cast<cudaStream_t>(stream);
    if (d->dtype == SPL_DTYPE_F32)
      interior_impl<float>(*d, q, k, head_offset, local_heads, softmax_out, dropout_mask, dropout_out, st);
    else
      interior_impl<bf16>(*d, q, k, head_offset, local_heads, softmax_out, dropout_mask, dropout_out, st);
  });
}

int spl_all_gather(const void* const* shards, int t, const int64_t* shape, int ndim, int axis,
                   int dtype, void* out, int64_t log[12], int tag, void* stream) {
  return bguard([&] {
    using namespace spl;
    rank_ptrs(shards, t, "all_gather");
    require(out != nullptr && shape != nullptr, "null buffer");
    const AxisBlocks blk = axis_blocks(shape, ndim, axis);
    const size_t es = esize(dtype);
    auto st = static_cast<cudaStream_t>(stream);
    const size_t width = es * (size_t)(blk.axis * blk.inner);
    for (int r = 0; r < t && width > 0 && blk.outer > 0; ++r) {
      // concat (tensor.cpp:169-203): part r lands at axis offset r·piece of every outer block
      SPL_CUDA(cudaMemcpy2DAsync(static_cast<char*>(out) + (size_t)r * width, width * (size_t)t,
                                 shards[r], width, width, (size_t)blk.outer,
                                 cudaMemcpyDeviceToDevice, st));
    }
    log_ring(log, tag, 0, blk.outer * blk.axis * blk.inner * t, t, 1);
  });
}

int spl_reduce_scatter(const void* const* partials, int t, const int64_t* shape, int ndim,
                       int axis, int dtype, void* const* out, int64_t log[12], int tag,
                       void* stream) {
  return bguard([&] {
    using namespace spl;
    RankPtrs in = rank_ptrs(partials, t, "reduce_scatter");
    require(out != nullptr && shape != nullptr, "null buffer");
    const AxisBlocks blk = axis_blocks(shape, ndim, axis);
    // split (tensor.cpp:212-214)
    if (blk.axis % t != 0) raise(SPL_EINVAL, "split axis not divisible by part count");
    const int64_t piece = blk.axis / t;
    const int64_t n = blk.outer * piece * blk.inner;
    auto st = static_cast<cudaStream_t>(stream);
    for (int r = 0; r < t; ++r) {
      require(out[r] != nullptr, "null output shard");
      sum_dispatch(dtype, in, t, out[r], n, piece, blk.inner, blk.axis, r * piece, st);
    }
    log_ring(log, tag, 1, blk.outer * blk.axis * blk.inner, t, 1);
  });
}

int spl_all_reduce(const void* const* partials, int t, const int64_t* shape, int ndim, int dtype,
                   void* out, int64_t log[12], int tag, void* stream) {
  return bguard([&] {
    using namespace spl;
    RankPtrs in = rank_ptrs(partials, t, "all_reduce");
    require(out != nullptr && (shape != nullptr || ndim == 0), "null buffer");
    int64_t n = 1;
    for (int i = 0; i < ndim; ++i) {
      require(shape[i] >= 0, "negative tensor dimension");
      n *= shape[i];
    }
    sum_dispatch(dtype, in, t, out, n, n, 1, n, 0, static_cast<cudaStream_t>(stream));
    log_ring(log, tag, 2, n, t, 2);
  });
}

}  // extern "C"
