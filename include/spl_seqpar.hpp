// spl_seqpar.hpp — header-only C++ facade over the C ABI (spl.h) with the reference's seqpar
// signatures, so code written against actplan::seqpar (block.hpp:28-174) switches by changing
// the namespace: `namespace seqpar = spl::seqpar;`.
//
//   reference (actplan::seqpar)                         facade (spl::seqpar)
//   BlockConfig                 block.hpp:28-42         BlockConfig (+ recompute, SP, dtype)
//   LayerParams::random/zeros   block.hpp:47-59         LayerParams::random/zeros (host fp64)
//   seqpar_block_forward        block.hpp:158-160       seqpar_block_forward  -> GPU layer
//   seqpar_block_backward       block.hpp:173-174       seqpar_block_backward -> GPU layer
//   ActivationLedger            block.hpp:61-73         ActivationLedger (+ physical bytes)
//   CommLog                     collectives.hpp:30-52   CommLog
//   per_layer_bytes             activation_memory.hpp:83 per_layer_bytes
//   layer_component_breakdown   activation_memory.cpp:84 layer_component_breakdown
//   percent_of_baseline         activation_memory.cpp:195 percent_of_baseline (num/den)
//   total_first_stage_bytes     activation_memory.cpp:119 total_first_stage_bytes
//   layer_comm_bytes_tensor_*   collectives.cpp:75-87   layer_comm_bytes_tensor_parallel/_sequence
// Errors: std::invalid_argument / std::domain_error exactly where the reference throws them.
// Tensors are host fp64 (as in the reference); device buffers are managed here with the CUDA
// runtime; the layer computes in fp32 (exact) or bf16 on the GPU.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "spl.h"

namespace spl::seqpar {

inline void check(int rc) {
  if (rc == SPL_OK) return;
  const std::string msg = spl_last_error();
  if (rc == SPL_EINVAL || rc == SPL_ESTATE) throw std::invalid_argument(msg);
  if (rc == SPL_EDOMAIN) throw std::domain_error(msg);
  throw std::runtime_error(msg);
}

class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(std::vector<int64_t> shape) : shape_(std::move(shape)) {
    int64_t n = 1;
    for (auto d : shape_) {
      if (d < 0) throw std::invalid_argument("negative tensor dimension");
      n *= d;
    }
    data_.assign((size_t)n, 0.0);
  }
  const std::vector<int64_t>& shape() const { return shape_; }
  int64_t dim(size_t i) const { return shape_.at(i); }
  int64_t numel() const { return (int64_t)data_.size(); }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  double& operator[](int64_t i) { return data_[(size_t)i]; }
  double operator[](int64_t i) const { return data_[(size_t)i]; }
  bool same_shape(const Tensor& o) const { return shape_ == o.shape_; }

 private:
  std::vector<int64_t> shape_;
  std::vector<double> data_;
};

enum class RecomputeKind { None = SPL_RECOMPUTE_NONE, Full = SPL_RECOMPUTE_FULL,
                           Selective = SPL_RECOMPUTE_SELECTIVE };
enum class DType { F32 = SPL_DTYPE_F32, BF16 = SPL_DTYPE_BF16 };

struct BlockConfig {
  int64_t heads = 0, hidden = 0, seq = 0, batch = 0;
  double dropout_p = 0.0;
  bool causal = false;
  uint64_t seed = 42;
  uint32_t layer_index = 0, microbatch = 1;
  double layer_norm_eps = 1e-5;
  // execution choices (not in the reference BlockConfig; defaults = the reference harness)
  RecomputeKind recompute = RecomputeKind::None;
  bool sequence_parallel = true;
  DType dtype = DType::F32;
  int device = 0;
  int64_t head_dim() const { return hidden / heads; }
};

// splitmix64 counter RNG (rng.cpp:22-37), host side, for LayerParams::random.
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t hash_counter(uint64_t key, uint64_t i) {
  return mix64(mix64(key) ^ mix64(i + 0x632be59bd9b4e019ULL));
}
inline double uniform01(uint64_t key, uint64_t i) {
  return (double)(hash_counter(key, i) >> 11) * 0x1.0p-53;
}
inline Tensor random_uniform(uint64_t key, std::vector<int64_t> shape, double lo, double hi) {
  Tensor t(std::move(shape));
  for (int64_t i = 0; i < t.numel(); ++i) t[i] = lo + (hi - lo) * uniform01(key, (uint64_t)i);
  return t;
}

struct LayerParams {
  Tensor wq, wk, wv, bq, bk, bv, wo, bo, w1, b1, w2, b2, ln1_gain, ln1_bias, ln2_gain, ln2_bias;

  std::vector<Tensor*> all() {
    return {&wq, &wk, &wv, &bq, &bk, &bv, &wo, &bo, &w1, &b1, &w2, &b2,
            &ln1_gain, &ln1_bias, &ln2_gain, &ln2_bias};
  }
  std::vector<const Tensor*> all() const {
    return {&wq, &wk, &wv, &bq, &bk, &bv, &wo, &bo, &w1, &b1, &w2, &b2,
            &ln1_gain, &ln1_bias, &ln2_gain, &ln2_bias};
  }
  static std::vector<std::vector<int64_t>> shapes(int64_t h) {
    return {{h, h}, {h, h}, {h, h}, {h}, {h}, {h}, {h, h}, {h}, {h, 4 * h}, {4 * h},
            {4 * h, h}, {h}, {h}, {h}, {h}, {h}};
  }
  // block.cpp:234-265
  static LayerParams random(const BlockConfig& cfg, uint64_t seed) {
    const int64_t h = cfg.hidden;
    const double ws = 1.0 / std::sqrt((double)h);
    static const bool weight[16] = {1, 1, 1, 0, 0, 0, 1, 0, 1, 0, 1, 0, 0, 0, 0, 0};
    LayerParams p;
    auto sh = shapes(h);
    auto ts = p.all();
    for (int i = 0; i < 16; ++i)
      *ts[i] = weight[i] ? random_uniform(hash_counter(seed, (uint64_t)(i + 1)), sh[i], -ws, ws)
                         : random_uniform(hash_counter(seed, (uint64_t)(i + 1)), sh[i], -0.1, 0.1);
    for (int64_t i = 0; i < h; ++i) {
      p.ln1_gain[i] += 1.0;
      p.ln2_gain[i] += 1.0;
    }
    return p;
  }
  static LayerParams zeros(const BlockConfig& cfg) {  // block.cpp:267-291
    const int64_t h = cfg.hidden;
    LayerParams p;
    auto sh = shapes(h);
    auto ts = p.all();
    for (int i = 0; i < 16; ++i) *ts[i] = Tensor(sh[i]);
    for (int64_t i = 0; i < h; ++i) p.ln1_gain[i] = p.ln2_gain[i] = 1.0;
    return p;
  }
  std::vector<double> packed() const {
    std::vector<double> v;
    for (const Tensor* t : all()) v.insert(v.end(), t->data(), t->data() + t->numel());
    return v;
  }
  static LayerParams unpack(int64_t h, const std::vector<double>& v) {
    LayerParams p;
    auto sh = shapes(h);
    auto ts = p.all();
    size_t off = 0;
    for (int i = 0; i < 16; ++i) {
      *ts[i] = Tensor(sh[i]);
      std::memcpy(ts[i]->data(), v.data() + off, sizeof(double) * (size_t)ts[i]->numel());
      off += (size_t)ts[i]->numel();
    }
    return p;
  }
};

struct LedgerEntry {
  std::string name;
  int64_t elements = 0, bytes = 0, physical_bytes = 0;
};
struct ActivationLedger {
  std::vector<LedgerEntry> entries;
  int64_t total_bytes() const {
    int64_t t = 0;
    for (auto& e : entries) t += e.bytes;
    return t;
  }
};
struct CommCounters {
  int64_t all_gathers = 0, reduce_scatters = 0, all_reduces = 0, ring_elements = 0;
};
struct CommLog {
  CommCounters schedule, regather, grad_sync, recompute;
};

namespace detail {
struct Handle {
  spl_handle* h = nullptr;
  std::vector<void*> dev;
  ~Handle() {
    for (void* p : dev) cudaFree(p);
    if (h) spl_destroy(h);
  }
};
inline void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}
inline uint16_t to_bf16(float f) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
inline double from_bf16(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
inline std::vector<char> host_to_dtype(const Tensor& t, DType dt) {
  std::vector<char> out((size_t)t.numel() * (dt == DType::F32 ? 4 : 2));
  for (int64_t i = 0; i < t.numel(); ++i) {
    if (dt == DType::F32) {
      const float f = (float)t[i];
      std::memcpy(out.data() + 4 * i, &f, 4);
    } else {
      const uint16_t b = to_bf16((float)t[i]);
      std::memcpy(out.data() + 2 * i, &b, 2);
    }
  }
  return out;
}
inline Tensor dtype_to_host(const std::vector<char>& v, std::vector<int64_t> shape, DType dt) {
  Tensor t(std::move(shape));
  for (int64_t i = 0; i < t.numel(); ++i) {
    if (dt == DType::F32) {
      float f;
      std::memcpy(&f, v.data() + 4 * i, 4);
      t[i] = f;
    } else {
      uint16_t b;
      std::memcpy(&b, v.data() + 2 * i, 2);
      t[i] = from_bf16(b);
    }
  }
  return t;
}
}  // namespace detail

struct SeqparForward {
  int64_t t = 1;
  BlockConfig cfg;
  std::vector<Tensor> y_shards;
  std::vector<ActivationLedger> ledgers;
  CommLog comm;
  std::shared_ptr<detail::Handle> layer;  // saved state lives on the device
};
struct SeqparBackward {
  std::vector<Tensor> dx_shards;
  LayerParams param_grads;
  std::vector<Tensor> w1_grad_shards;
  CommLog comm;
};

inline CommLog read_comm(spl_handle* h) {
  int64_t c[16];
  check(spl_comm_log(h, c));
  CommLog l;
  CommCounters* tags[4] = {&l.schedule, &l.regather, &l.grad_sync, &l.recompute};
  for (int i = 0; i < 4; ++i) *tags[i] = {c[4 * i], c[4 * i + 1], c[4 * i + 2], c[4 * i + 3]};
  return l;
}

// seqpar_block_forward (block.cpp:512-602)
inline SeqparForward seqpar_block_forward(const std::vector<Tensor>& x_shards,
                                          const LayerParams& params, int64_t t,
                                          const BlockConfig& cfg) {
  if (t < 1) throw std::invalid_argument("t must be >= 1");
  if ((int64_t)x_shards.size() != t) throw std::invalid_argument("expected one input shard per rank");
  spl_layer_desc d;
  spl_desc_default(&d);
  d.heads = cfg.heads; d.hidden = cfg.hidden; d.seq = cfg.seq; d.batch = cfg.batch;
  d.dropout_p = cfg.dropout_p; d.causal = cfg.causal; d.seed = cfg.seed;
  d.layer_index = cfg.layer_index; d.microbatch = cfg.microbatch; d.ln_eps = cfg.layer_norm_eps;
  d.recompute = (int)cfg.recompute; d.sequence_parallel = cfg.sequence_parallel;
  d.dtype = (int)cfg.dtype;
  auto H = std::make_shared<detail::Handle>();
  check(spl_create_local(&d, cfg.device, (int)t, &H->h));
  const int64_t rows = cfg.sequence_parallel ? cfg.seq / t : cfg.seq;
  const std::vector<int64_t> shard{rows, cfg.batch, cfg.hidden};
  for (const Tensor& x : x_shards)
    if (x.shape() != shard) throw std::invalid_argument("input shard must be {s/t, b, h}");
  auto packed = params.packed();
  check(spl_load_params(H->h, packed.data()));
  const size_t bytes = (size_t)(rows * cfg.batch * cfg.hidden) * (cfg.dtype == DType::F32 ? 4 : 2);
  std::vector<const void*> xs;
  std::vector<void*> ys;
  for (int64_t r = 0; r < t; ++r) {
    void *px, *py;
    detail::cuda(cudaMalloc(&px, bytes));
    detail::cuda(cudaMalloc(&py, bytes));
    H->dev.push_back(px);
    H->dev.push_back(py);
    auto hx = detail::host_to_dtype(x_shards[(size_t)r], cfg.dtype);
    detail::cuda(cudaMemcpy(px, hx.data(), bytes, cudaMemcpyHostToDevice));
    xs.push_back(px);
    ys.push_back(py);
  }
  check(spl_forward(H->h, xs.data(), ys.data()));
  detail::cuda(cudaDeviceSynchronize());
  SeqparForward f;
  f.t = t;
  f.cfg = cfg;
  for (int64_t r = 0; r < t; ++r) {
    std::vector<char> hy(bytes);
    detail::cuda(cudaMemcpy(hy.data(), ys[(size_t)r], bytes, cudaMemcpyDeviceToHost));
    f.y_shards.push_back(detail::dtype_to_host(hy, shard, cfg.dtype));
    spl_ledger_entry e[32];
    int n = 32;
    check(spl_ledger(H->h, (int)r, e, &n));
    ActivationLedger L;
    for (int i = 0; i < n; ++i) L.entries.push_back({e[i].name, e[i].elements, e[i].bytes, e[i].physical_bytes});
    f.ledgers.push_back(L);
  }
  f.comm = read_comm(H->h);
  f.layer = H;
  return f;
}

// seqpar_block_backward (block.cpp:622-749)
inline SeqparBackward seqpar_block_backward(const std::vector<Tensor>& dy_shards,
                                            const SeqparForward& fwd, const LayerParams&) {
  if (!fwd.layer || fwd.y_shards.empty()) throw std::invalid_argument("missing saved forward state");
  if ((int64_t)dy_shards.size() != fwd.t) throw std::invalid_argument("expected one gradient shard per rank");
  const BlockConfig& cfg = fwd.cfg;
  for (size_t r = 0; r < dy_shards.size(); ++r)
    if (!dy_shards[r].same_shape(fwd.y_shards[r])) throw std::invalid_argument("dy shard shape mismatch");
  spl_handle* h = fwd.layer->h;
  check(spl_comm_log_reset(h));
  const std::vector<int64_t> shard = fwd.y_shards[0].shape();
  const size_t bytes = (size_t)fwd.y_shards[0].numel() * (cfg.dtype == DType::F32 ? 4 : 2);
  std::vector<const void*> ds;
  std::vector<void*> dx;
  for (int64_t r = 0; r < fwd.t; ++r) {
    void *pd, *px;
    detail::cuda(cudaMalloc(&pd, bytes));
    detail::cuda(cudaMalloc(&px, bytes));
    fwd.layer->dev.push_back(pd);
    fwd.layer->dev.push_back(px);
    auto hd = detail::host_to_dtype(dy_shards[(size_t)r], cfg.dtype);
    detail::cuda(cudaMemcpy(pd, hd.data(), bytes, cudaMemcpyHostToDevice));
    ds.push_back(pd);
    dx.push_back(px);
  }
  check(spl_backward(h, ds.data(), dx.data()));
  detail::cuda(cudaDeviceSynchronize());
  SeqparBackward b;
  for (int64_t r = 0; r < fwd.t; ++r) {
    std::vector<char> hx(bytes);
    detail::cuda(cudaMemcpy(hx.data(), dx[(size_t)r], bytes, cudaMemcpyDeviceToHost));
    b.dx_shards.push_back(detail::dtype_to_host(hx, shard, cfg.dtype));
    Tensor w1({cfg.hidden, 4 * cfg.hidden / fwd.t});
    check(spl_get_w1_grad_shard(h, (int)r, w1.data()));
    b.w1_grad_shards.push_back(std::move(w1));
  }
  std::vector<double> g((size_t)(12 * cfg.hidden * cfg.hidden + 13 * cfg.hidden));
  check(spl_get_grads(h, g.data()));
  b.param_grads = LayerParams::unpack(cfg.hidden, g);
  b.comm = read_comm(h);
  return b;
}

// per_layer_bytes (activation_memory.cpp:79-82)
inline int64_t per_layer_bytes(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t,
                               RecomputeKind kind, bool sequence_parallel, int64_t act = 2,
                               int64_t mask = 1) {
  int64_t out = 0;
  check(spl_per_layer_bytes(a, h, s, b, t, (int)kind, sequence_parallel ? 1 : 0, act, mask, &out));
  return out;
}

// layer_component_breakdown (activation_memory.cpp:84-104), serial layer
struct LayerMemoryBreakdown {
  int64_t attention = 0, mlp = 0, layer_norms = 0, total = 0;
};
inline LayerMemoryBreakdown layer_component_breakdown(int64_t a, int64_t h, int64_t s, int64_t b,
                                                      int64_t act = 2, int64_t mask = 1) {
  int64_t o[4];
  check(spl_layer_component_breakdown(a, h, s, b, act, mask, o));
  return {o[0], o[1], o[2], o[3]};
}

// percent_of_baseline (activation_memory.cpp:195-200) as an exact fraction
struct Fraction {
  int64_t num = 0, den = 1;
};
inline Fraction percent_of_baseline(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t,
                                    RecomputeKind kind, bool sequence_parallel, int64_t act = 2,
                                    int64_t mask = 1) {
  Fraction f;
  check(spl_percent_of_baseline(a, h, s, b, t, (int)kind, sequence_parallel ? 1 : 0, act, mask,
                                &f.num, &f.den));
  return f;
}

// total_first_stage_bytes (activation_memory.cpp:112-123): L layers, p stages, m interleave
inline int64_t total_first_stage_bytes(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t,
                                       RecomputeKind kind, bool sequence_parallel, int64_t layers,
                                       int64_t pipeline = 1, int64_t interleave = 1,
                                       int64_t act = 2, int64_t mask = 1) {
  int64_t out = 0;
  check(spl_total_first_stage_bytes(a, h, s, b, t, (int)kind, sequence_parallel ? 1 : 0, layers,
                                    pipeline, interleave, act, mask, &out));
  return out;
}

// layer_comm_bytes_tensor_parallel / _tensor_sequence (collectives.cpp:75-87)
inline int64_t layer_comm_bytes_tensor_parallel(int64_t seq, int64_t batch, int64_t hidden,
                                                int64_t t, int64_t elem_bytes) {
  int64_t out = 0;
  check(spl_layer_comm_bytes(seq, batch, hidden, t, elem_bytes, 0, &out));
  return out;
}
inline int64_t layer_comm_bytes_tensor_sequence(int64_t seq, int64_t batch, int64_t hidden,
                                                int64_t t, int64_t elem_bytes) {
  int64_t out = 0;
  check(spl_layer_comm_bytes(seq, batch, hidden, t, elem_bytes, 1, &out));
  return out;
}

}  // namespace spl::seqpar
