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
//   seqpar_block_forward(RankShardedTensor) block.hpp:158-162 same overload
//   reference_block_forward/_backward block.hpp:121-130 -> the t = 1 GPU layer
//   attention_interior          block.hpp:100-101       attention_interior -> GPU kernel
//   all_gather/reduce_scatter/all_reduce collectives.hpp:57-62 -> device rank-ordered ops (fp64)
//   concat/split/slice_part, RankShardedTensor tensor.hpp:66-89 (host helpers)
//   RecomputeStrategy::parse/name config.hpp:53-67, config.cpp:36-84
// Errors: std::invalid_argument / std::domain_error exactly where the reference throws them.
// Tensors are host fp64 (as in the reference); device buffers are managed here with the CUDA
// runtime; the layer computes in fp32 (exact) or bf16 on the GPU.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
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

// RecomputeStrategy (config.hpp:53-67): parse / name restate config.cpp:36-84, same messages.
struct RecomputeStrategy {
  RecomputeKind kind = RecomputeKind::None;
  bool sequence_parallel = false;
  bool microbatch_level = false;

  static RecomputeStrategy parse(std::string_view spec) {
    RecomputeStrategy out;
    bool have_kind = false;
    std::string_view rest = spec;
    while (!rest.empty()) {
      const auto pos = rest.find('+');
      const std::string_view tok = rest.substr(0, pos);
      rest = pos == std::string_view::npos ? std::string_view{} : rest.substr(pos + 1);
      if (tok == "none" || tok == "full" || tok == "selective") {
        if (have_kind)
          throw std::invalid_argument("strategy '" + std::string(spec) +
                                      "' names more than one recompute kind");
        have_kind = true;
        out.kind = tok == "none" ? RecomputeKind::None
                                 : tok == "full" ? RecomputeKind::Full : RecomputeKind::Selective;
      } else if (tok == "seq") {
        out.sequence_parallel = true;
      } else if (tok == "mblevel") {
        out.microbatch_level = true;
      } else {
        throw std::invalid_argument("unknown strategy token '" + std::string(tok) +
                                    "' (expected none|full|selective with optional +seq, +mblevel)");
      }
    }
    if (!have_kind)
      throw std::invalid_argument("strategy '" + std::string(spec) +
                                  "' must name one of none|full|selective");
    if (out.microbatch_level && out.kind == RecomputeKind::None)
      throw std::invalid_argument("'none+mblevel' is not a strategy: the microbatch window needs "
                                  "a full or selective base to checkpoint with");
    return out;
  }
  std::string name() const {
    std::string out = kind == RecomputeKind::None ? "none"
                      : kind == RecomputeKind::Full ? "full" : "selective";
    if (sequence_parallel) out += "+seq";
    if (microbatch_level) out += "+mblevel";
    return out;
  }
  bool operator==(const RecomputeStrategy&) const = default;
};

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


// ---- host tensor helpers with the reference's axis semantics (tensor.cpp:127-259)
inline bool bit_equal(const Tensor& a, const Tensor& b) {
  return a.same_shape(b) && std::memcmp(a.data(), b.data(), sizeof(double) * (size_t)a.numel()) == 0;
}
inline double max_abs_diff(const Tensor& a, const Tensor& b) {
  if (!a.same_shape(b)) throw std::invalid_argument("max_abs_diff: shape mismatch");
  double m = 0.0;
  for (int64_t i = 0; i < a.numel(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}
namespace detail {
struct AxisBlocks {
  int64_t outer = 1, axis = 1, inner = 1;
};
inline AxisBlocks axis_blocks(const std::vector<int64_t>& shape, size_t axis) {
  if (axis >= shape.size()) throw std::invalid_argument("axis out of range");
  AxisBlocks b;
  for (size_t i = 0; i < shape.size(); ++i) {
    if (i < axis) b.outer *= shape[i];
    else if (i == axis) b.axis = shape[i];
    else b.inner *= shape[i];
  }
  return b;
}
}  // namespace detail
inline Tensor concat(std::span<const Tensor> parts, size_t axis) {
  if (parts.empty()) throw std::invalid_argument("concat: no parts");
  std::vector<int64_t> shape = parts[0].shape();
  int64_t total = 0;
  for (const Tensor& p : parts) {
    if (p.shape().size() != shape.size()) throw std::invalid_argument("concat: rank mismatch");
    for (size_t i = 0; i < shape.size(); ++i)
      if (i != axis && p.shape()[i] != shape[i])
        throw std::invalid_argument("concat: shape mismatch off the concat axis");
    total += p.shape().at(axis);
  }
  shape[axis] = total;
  Tensor out(shape);
  const auto ob = detail::axis_blocks(shape, axis);
  int64_t off = 0;
  for (const Tensor& p : parts) {
    const auto ib = detail::axis_blocks(p.shape(), axis);
    for (int64_t o = 0; o < ib.outer; ++o)
      std::memcpy(out.data() + (o * ob.axis + off) * ob.inner, p.data() + o * ib.axis * ib.inner,
                  sizeof(double) * (size_t)(ib.axis * ib.inner));
    off += ib.axis;
  }
  return out;
}
inline Tensor slice_part(const Tensor& x, size_t axis, int64_t parts, int64_t index) {
  const auto b = detail::axis_blocks(x.shape(), axis);
  if (parts < 1 || b.axis % parts != 0) throw std::invalid_argument("split axis not divisible by part count");
  if (index < 0 || index >= parts) throw std::invalid_argument("slice index out of range");
  const int64_t piece = b.axis / parts;
  std::vector<int64_t> shape = x.shape();
  shape[axis] = piece;
  Tensor out(shape);
  for (int64_t o = 0; o < b.outer; ++o)
    std::memcpy(out.data() + o * piece * b.inner, x.data() + (o * b.axis + index * piece) * b.inner,
                sizeof(double) * (size_t)(piece * b.inner));
  return out;
}
inline std::vector<Tensor> split(const Tensor& x, size_t axis, int64_t parts) {
  std::vector<Tensor> out;
  for (int64_t r = 0; r < parts; ++r) out.push_back(slice_part(x, axis, parts, r));
  return out;
}

enum class ShardAxis { Sequence, Hidden, Replicated };

// RankShardedTensor (tensor.hpp:80-89, tensor.cpp:227-259)
struct RankShardedTensor {
  std::vector<Tensor> shards;
  ShardAxis axis = ShardAxis::Replicated;
  std::vector<int64_t> logical_shape;

  static RankShardedTensor from_full(const Tensor& full, ShardAxis axis, size_t axis_index,
                                     int64_t ranks) {
    RankShardedTensor out;
    out.axis = axis;
    out.logical_shape = full.shape();
    if (axis == ShardAxis::Replicated) out.shards.assign((size_t)ranks, full);
    else out.shards = split(full, axis_index, ranks);
    return out;
  }
  Tensor to_full(size_t axis_index) const {
    if (axis == ShardAxis::Replicated) return shards.at(0);
    return concat(shards, axis_index);
  }
  void check() const {
    if (shards.empty()) throw std::invalid_argument("sharded tensor has no shards");
    for (const Tensor& s : shards)
      if (!s.same_shape(shards[0])) throw std::invalid_argument("shard shapes differ across ranks");
    if (axis == ShardAxis::Replicated)
      for (const Tensor& s : shards)
        if (!bit_equal(s, shards[0]))
          throw std::invalid_argument("replicated tensor has diverging shards");
  }
};

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
  uint64_t params_hash = 0;               // of the LayerParams the forward ran with
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

namespace detail {
inline spl_layer_desc make_desc(const BlockConfig& cfg) {
  spl_layer_desc d;
  spl_desc_default(&d);
  d.heads = cfg.heads; d.hidden = cfg.hidden; d.seq = cfg.seq; d.batch = cfg.batch;
  d.dropout_p = cfg.dropout_p; d.causal = cfg.causal; d.seed = cfg.seed;
  d.layer_index = cfg.layer_index; d.microbatch = cfg.microbatch; d.ln_eps = cfg.layer_norm_eps;
  d.recompute = (int)cfg.recompute; d.sequence_parallel = cfg.sequence_parallel;
  d.dtype = (int)cfg.dtype;
  return d;
}
// FNV-1a over the packed parameter bytes: detects a backward called with other parameters.
inline uint64_t hash_params(const std::vector<double>& v) {
  uint64_t h = 1469598103934665603ULL;
  const unsigned char* p = reinterpret_cast<const unsigned char*>(v.data());
  for (size_t i = 0; i < v.size() * sizeof(double); ++i) h = (h ^ p[i]) * 1099511628211ULL;
  return h;
}
}  // namespace detail

// seqpar_block_forward (block.cpp:512-602)
inline SeqparForward seqpar_block_forward(const std::vector<Tensor>& x_shards,
                                          const LayerParams& params, int64_t t,
                                          const BlockConfig& cfg) {
  if (t < 1) throw std::invalid_argument("t must be >= 1");
  if ((int64_t)x_shards.size() != t) throw std::invalid_argument("expected one input shard per rank");
  const spl_layer_desc d = detail::make_desc(cfg);
  auto H = std::make_shared<detail::Handle>();
  check(spl_create_local(&d, cfg.device, (int)t, &H->h));
  const int64_t rows = cfg.sequence_parallel ? cfg.seq / t : cfg.seq;
  const std::vector<int64_t> shard{rows, cfg.batch, cfg.hidden};
  for (const Tensor& x : x_shards)
    if (x.shape() != shard) throw std::invalid_argument("input shard must be {s/t, b, h}");
  auto packed = params.packed();
  check(spl_load_params(H->h, packed.data()));
  const uint64_t phash = detail::hash_params(packed);
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
  f.params_hash = phash;
  return f;
}

// seqpar_block_backward (block.cpp:622-749)
// The backward GEMMs use `params` (block.cpp:639-640: shard_params of the argument), so when
// they differ from the forward's the device weights are reloaded first. Under full
// recomputation the device would then also re-run the forward with them, which the reference
// never does (it keeps the forward's activations), so that combination is rejected.
inline SeqparBackward seqpar_block_backward(const std::vector<Tensor>& dy_shards,
                                            const SeqparForward& fwd, const LayerParams& params) {
  if (!fwd.layer || fwd.y_shards.empty()) throw std::invalid_argument("missing saved forward state");
  if ((int64_t)dy_shards.size() != fwd.t) throw std::invalid_argument("expected one gradient shard per rank");
  const BlockConfig& cfg = fwd.cfg;
  for (size_t r = 0; r < dy_shards.size(); ++r)
    if (!dy_shards[r].same_shape(fwd.y_shards[r])) throw std::invalid_argument("dy shard shape mismatch");
  spl_handle* h = fwd.layer->h;
  {
    const auto packed = params.packed();
    if ((int64_t)packed.size() != 12 * cfg.hidden * cfg.hidden + 13 * cfg.hidden)
      throw std::invalid_argument("params do not match the forward's hidden size");
    if (detail::hash_params(packed) != fwd.params_hash) {
      if (cfg.recompute == RecomputeKind::Full)
        throw std::invalid_argument("full recomputation re-runs the forward: backward params must "
                                    "be the forward's");
      check(spl_load_params(h, packed.data()));
    }
  }
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

// seqpar_block_forward(const RankShardedTensor&, params, cfg) (block.hpp:158-162, block.cpp:604-613)
inline SeqparForward seqpar_block_forward(const RankShardedTensor& x, const LayerParams& params,
                                          const BlockConfig& cfg) {
  if (x.axis != ShardAxis::Sequence)
    throw std::invalid_argument("layer input must be sharded along the sequence axis");
  x.check();
  return seqpar_block_forward(x.shards, params, (int64_t)x.shards.size(), cfg);
}

// ReferenceForward / BlockGrads (block.hpp:104-130): the single-rank oracle. On the GPU it is
// the t = 1 layer — the reference's own t = 1 seqpar path is bit-identical to it
// (test_seqpar.cpp:161-168), so one implementation serves both.
struct ReferenceForward {
  Tensor y;
  ActivationLedger ledger;
  BlockConfig cfg;
  std::shared_ptr<detail::Handle> layer;
  uint64_t params_hash = 0;

  // A saved tensor of the forward by ledger name (block.hpp:110-118 members: "query", "key",
  // "value", "attn_proj_input", "attn_dropout_mask", "gelu_input", …), read back in fp64.
  Tensor saved(const std::string& name) const {
    if (!layer) throw std::invalid_argument("missing saved forward state");
    for (const LedgerEntry& e : ledger.entries) {
      if (e.name != name) continue;
      Tensor out(std::vector<int64_t>{e.elements});
      check(spl_get_saved(layer->h, 0, name.c_str(), out.data(), e.elements));
      return out;
    }
    throw std::invalid_argument("no saved tensor named " + name);
  }
  Tensor attn_dropout_mask() const { return saved("attn_dropout_mask"); }
  Tensor mlp_dropout_mask() const { return saved("mlp_dropout_mask"); }
};
struct BlockGrads {
  LayerParams params;
  Tensor dx;
};

// reference_block_forward (block.cpp:419-456)
inline ReferenceForward reference_block_forward(const Tensor& x, const LayerParams& params,
                                                const BlockConfig& cfg) {
  if (x.shape() != std::vector<int64_t>{cfg.seq, cfg.batch, cfg.hidden})
    throw std::invalid_argument("reference_block_forward: input must be {s, b, h}");
  if (cfg.heads <= 0 || cfg.hidden % cfg.heads != 0)
    throw std::invalid_argument("hidden not divisible by heads");
  BlockConfig c = cfg;
  c.sequence_parallel = true;  // one rank: its sequence shard is the whole {s, b, h}
  SeqparForward f = seqpar_block_forward(std::vector<Tensor>{x}, params, 1, c);
  ReferenceForward r;
  r.y = std::move(f.y_shards[0]);
  r.ledger = std::move(f.ledgers[0]);
  r.cfg = c;
  r.layer = f.layer;
  r.params_hash = f.params_hash;
  return r;
}

// reference_block_backward (block.cpp:458-510)
inline BlockGrads reference_block_backward(const Tensor& dy, const ReferenceForward& fwd,
                                           const LayerParams& params) {
  if (!fwd.layer) throw std::invalid_argument("missing saved forward state");
  if (!dy.same_shape(fwd.y)) throw std::invalid_argument("dy shape mismatch");
  SeqparForward f;
  f.t = 1;
  f.cfg = fwd.cfg;
  f.y_shards = {fwd.y};
  f.layer = fwd.layer;
  f.params_hash = fwd.params_hash;
  SeqparBackward b = seqpar_block_backward(std::vector<Tensor>{dy}, f, params);
  return BlockGrads{std::move(b.param_grads), std::move(b.dx_shards[0])};
}

// AttentionInterior (block.hpp:91-97) and attention_interior(q, k, cfg, head_offset,
// local_heads) (block.hpp:100-101, block.cpp:381-417) on the GPU kernel, in cfg.dtype.
struct AttentionInterior {
  Tensor softmax_out, dropout_mask, dropout_out;  // {local_heads, b, s, s}
};
inline AttentionInterior attention_interior(const Tensor& q, const Tensor& k, const BlockConfig& cfg,
                                            int64_t head_offset, int64_t local_heads) {
  if (cfg.heads <= 0 || cfg.hidden % cfg.heads != 0)
    throw std::invalid_argument("hidden not divisible by heads");
  const int64_t lw = local_heads * cfg.head_dim();
  const std::vector<int64_t> qs{cfg.seq, cfg.batch, lw};
  if (q.shape() != qs || k.shape() != qs)
    throw std::invalid_argument("attention_interior: q and k must be {s, b, local_heads*hd}");
  const spl_layer_desc d = detail::make_desc(cfg);
  const size_t es = cfg.dtype == DType::F32 ? 4 : 2;
  const int64_t n = local_heads * cfg.batch * cfg.seq * cfg.seq;
  detail::cuda(cudaSetDevice(cfg.device));
  std::vector<void*> bufs(5, nullptr);
  struct Free {
    std::vector<void*>& b;
    ~Free() { for (void* p : b) cudaFree(p); }
  } guard{bufs};
  detail::cuda(cudaMalloc(&bufs[0], es * (size_t)q.numel()));
  detail::cuda(cudaMalloc(&bufs[1], es * (size_t)k.numel()));
  detail::cuda(cudaMalloc(&bufs[2], es * (size_t)n));
  detail::cuda(cudaMalloc(&bufs[3], (size_t)n));
  detail::cuda(cudaMalloc(&bufs[4], es * (size_t)n));
  auto hq = detail::host_to_dtype(q, cfg.dtype), hk = detail::host_to_dtype(k, cfg.dtype);
  detail::cuda(cudaMemcpy(bufs[0], hq.data(), hq.size(), cudaMemcpyHostToDevice));
  detail::cuda(cudaMemcpy(bufs[1], hk.data(), hk.size(), cudaMemcpyHostToDevice));
  check(spl_attention_interior_qk(&d, cfg.device, bufs[0], bufs[1], head_offset, local_heads,
                                  bufs[2], static_cast<uint8_t*>(bufs[3]), bufs[4], nullptr));
  detail::cuda(cudaDeviceSynchronize());
  const std::vector<int64_t> shape{local_heads, cfg.batch, cfg.seq, cfg.seq};
  std::vector<char> hs(es * (size_t)n), hd(es * (size_t)n), hm((size_t)n);
  detail::cuda(cudaMemcpy(hs.data(), bufs[2], hs.size(), cudaMemcpyDeviceToHost));
  detail::cuda(cudaMemcpy(hm.data(), bufs[3], hm.size(), cudaMemcpyDeviceToHost));
  detail::cuda(cudaMemcpy(hd.data(), bufs[4], hd.size(), cudaMemcpyDeviceToHost));
  AttentionInterior out{detail::dtype_to_host(hs, shape, cfg.dtype), Tensor(shape),
                        detail::dtype_to_host(hd, shape, cfg.dtype)};
  for (int64_t i = 0; i < n; ++i) out.dropout_mask[i] = hm[(size_t)i] ? 1.0 : 0.0;
  return out;
}

// Collectives over the simulated rank group (collectives.hpp:57-62): the shards go to the
// device in fp64 and the rank-ordered device sums are bit-identical to ordered_sum
// (collectives.cpp:30-38). CommTag maps to the CommLog fields like CommLog::by_tag.
enum class CommTag { Schedule = 0, Regather = 1, GradSync = 2 };
namespace detail {
inline void check_group(std::span<const Tensor> ts, const char* op) {
  if (ts.empty()) throw std::invalid_argument(std::string(op) + ": empty rank group");
  for (const Tensor& t : ts)
    if (!t.same_shape(ts[0])) throw std::invalid_argument(std::string(op) + ": shard shapes differ across ranks");
}
struct DevGroup {
  std::vector<void*> p;
  ~DevGroup() { for (void* q : p) cudaFree(q); }
  void* add(size_t bytes) {
    void* q = nullptr;
    cuda(cudaMalloc(&q, std::max<size_t>(bytes, 8)));
    p.push_back(q);
    return q;
  }
};
inline void merge_log(CommLog* log, const int64_t l[12]) {
  if (log == nullptr) return;
  CommCounters* c[3] = {&log->schedule, &log->regather, &log->grad_sync};
  for (int i = 0; i < 3; ++i) {
    c[i]->all_gathers += l[4 * i];
    c[i]->reduce_scatters += l[4 * i + 1];
    c[i]->all_reduces += l[4 * i + 2];
    c[i]->ring_elements += l[4 * i + 3];
  }
}
inline std::vector<const void*> upload(DevGroup& g, std::span<const Tensor> ts) {
  std::vector<const void*> v;
  for (const Tensor& t : ts) {
    void* q = g.add(sizeof(double) * (size_t)t.numel());
    cuda(cudaMemcpy(q, t.data(), sizeof(double) * (size_t)t.numel(), cudaMemcpyHostToDevice));
    v.push_back(q);
  }
  return v;
}
inline Tensor download(const void* p, std::vector<int64_t> shape) {
  Tensor t(std::move(shape));
  cuda(cudaMemcpy(t.data(), p, sizeof(double) * (size_t)t.numel(), cudaMemcpyDeviceToHost));
  return t;
}
}  // namespace detail

inline Tensor all_gather(std::span<const Tensor> shards, size_t axis, CommLog* log = nullptr,
                         CommTag tag = CommTag::Schedule) {
  detail::check_group(shards, "all_gather");
  std::vector<int64_t> shape = shards[0].shape();
  if (axis >= shape.size()) throw std::invalid_argument("axis out of range");
  detail::DevGroup g;
  auto in = detail::upload(g, shards);
  std::vector<int64_t> out_shape = shape;
  out_shape[axis] *= (int64_t)shards.size();
  void* out = g.add(sizeof(double) * (size_t)shards[0].numel() * shards.size());
  int64_t l[12] = {};
  check(spl_all_gather(in.data(), (int)shards.size(), shape.data(), (int)shape.size(), (int)axis,
                       SPL_DTYPE_F64, out, l, (int)tag, nullptr));
  detail::cuda(cudaDeviceSynchronize());
  detail::merge_log(log, l);
  return detail::download(out, out_shape);
}

inline std::vector<Tensor> reduce_scatter(std::span<const Tensor> partials, size_t axis,
                                          CommLog* log = nullptr, CommTag tag = CommTag::Schedule) {
  detail::check_group(partials, "reduce_scatter");
  std::vector<int64_t> shape = partials[0].shape();
  if (axis >= shape.size()) throw std::invalid_argument("axis out of range");
  const int64_t t = (int64_t)partials.size();
  if (shape[axis] % t != 0) throw std::invalid_argument("split axis not divisible by part count");
  detail::DevGroup g;
  auto in = detail::upload(g, partials);
  std::vector<void*> out;
  for (int64_t r = 0; r < t; ++r) out.push_back(g.add(sizeof(double) * (size_t)(partials[0].numel() / t)));
  int64_t l[12] = {};
  check(spl_reduce_scatter(in.data(), (int)t, shape.data(), (int)shape.size(), (int)axis,
                           SPL_DTYPE_F64, out.data(), l, (int)tag, nullptr));
  detail::cuda(cudaDeviceSynchronize());
  detail::merge_log(log, l);
  std::vector<int64_t> piece = shape;
  piece[axis] /= t;
  std::vector<Tensor> res;
  for (int64_t r = 0; r < t; ++r) res.push_back(detail::download(out[(size_t)r], piece));
  return res;
}

inline Tensor all_reduce(std::span<const Tensor> partials, CommLog* log = nullptr,
                         CommTag tag = CommTag::Schedule) {
  detail::check_group(partials, "all_reduce");
  std::vector<int64_t> shape = partials[0].shape();
  detail::DevGroup g;
  auto in = detail::upload(g, partials);
  void* out = g.add(sizeof(double) * (size_t)partials[0].numel());
  int64_t l[12] = {};
  check(spl_all_reduce(in.data(), (int)partials.size(), shape.data(), (int)shape.size(),
                       SPL_DTYPE_F64, out, l, (int)tag, nullptr));
  detail::cuda(cudaDeviceSynchronize());
  detail::merge_log(log, l);
  return detail::download(out, shape);
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
