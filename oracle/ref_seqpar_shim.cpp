// C entry layer over the reference's OWN seqpar harness — TEST INFRASTRUCTURE ONLY.
//
// oracle/Makefile `ref` compiles /root/reference/proj/core/src/seqpar/{tensor,block,
// collectives,rng}.cpp UNMODIFIED (against the Eigen/Boost stand-ins in oracle/shim/) together
// with this file into oracle/_ref/libref_seqpar.so. Nothing here re-implements the algorithm:
// every entry point converts flat fp64 buffers to actplan::seqpar::Tensor, calls the
// reference function named in its comment, and copies the result out. Used by
//   oracle/gen_layer_golden.py   -> tests/golden/layer_*.npz (committed fixtures)
//   tests/test_ref_golden.py     -> the C restatement (liboracle.so) vs the reference itself
//   bench.py --impl reference    -> the reference's own single-threaded CPU path, timed
// The product library (libspl.so) never links or loads it.
//
// Layouts match oracle/oracle.h: {s,b,h} row-major activations, LayerParams packed in
// named_tensors() order (block.cpp:293-298), interiors as {3, a, b, s, s}.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "actplan/seqpar/block.hpp"
#include "actplan/seqpar/collectives.hpp"
#include "actplan/seqpar/rng.hpp"
#include "actplan/seqpar/tensor.hpp"

using namespace actplan::seqpar;

namespace {

thread_local std::string g_err;

struct CfgC {  // == orc_block_cfg (oracle/oracle.h)
  std::int64_t heads, hidden, seq, batch;
  double dropout_p;
  std::int32_t causal;
  std::uint64_t seed;
  std::uint32_t layer_index, microbatch;
  double ln_eps;
};

struct CountersC {
  std::int64_t all_gathers, reduce_scatters, all_reduces, ring_elements;
};
struct CommLogC {
  CountersC schedule, regather, grad_sync;
};
struct LedgerC {
  std::int64_t elements[15];
  std::int64_t bytes[15];
};

BlockConfig to_cfg(const CfgC& c) {
  BlockConfig cfg;
  cfg.heads = c.heads;
  cfg.hidden = c.hidden;
  cfg.seq = c.seq;
  cfg.batch = c.batch;
  cfg.dropout_p = c.dropout_p;
  cfg.causal = c.causal != 0;
  cfg.seed = c.seed;
  cfg.layer_index = c.layer_index;
  cfg.microbatch = c.microbatch;
  cfg.layer_norm_eps = c.ln_eps;
  return cfg;
}

Tensor from_ptr(const double* p, std::vector<std::int64_t> shape) {
  Tensor t(std::move(shape));
  std::memcpy(t.data(), p, sizeof(double) * static_cast<std::size_t>(t.numel()));
  return t;
}

void to_ptr(const Tensor& t, double* p) {
  std::memcpy(p, t.data(), sizeof(double) * static_cast<std::size_t>(t.numel()));
}

std::int64_t big_to_i64(const actplan::BigInt& v) { return actplan::to_int64(v); }

void put_counters(const CommCounters& c, CountersC* out) {
  out->all_gathers = c.all_gathers;
  out->reduce_scatters = c.reduce_scatters;
  out->all_reduces = c.all_reduces;
  out->ring_elements = big_to_i64(c.ring_elements);
}

void put_log(const CommLog& log, CommLogC* out) {
  if (out == nullptr) return;
  put_counters(log.schedule, &out->schedule);
  put_counters(log.regather, &out->regather);
  put_counters(log.grad_sync, &out->grad_sync);
}

void put_ledger(const ActivationLedger& l, LedgerC* out) {
  if (out == nullptr) return;
  if (l.entries.size() != 15) throw std::logic_error("ledger entry count");
  for (std::size_t i = 0; i < 15; ++i) {
    out->elements[i] = l.entries[i].elements;
    out->bytes[i] = l.entries[i].bytes;
  }
}

// LayerParams <-> packed buffer in named_tensors() order.
LayerParams params_from(const BlockConfig& cfg, const double* packed) {
  LayerParams p = LayerParams::zeros(cfg);
  std::int64_t off = 0;
  for (auto& [name, tensor] : p.named_tensors()) {
    std::memcpy(tensor->data(), packed + off, sizeof(double) * static_cast<std::size_t>(tensor->numel()));
    off += tensor->numel();
  }
  return p;
}

void params_to(LayerParams& p, double* packed) {
  std::int64_t off = 0;
  for (auto& [name, tensor] : p.named_tensors()) {
    std::memcpy(packed + off, tensor->data(), sizeof(double) * static_cast<std::size_t>(tensor->numel()));
    off += tensor->numel();
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

void put_interior(const std::vector<AttentionInterior>& parts, double* out, std::int64_t full) {
  // out: {3, a, b, s, s}; rank r's {lh, b, s, s} block lands at head offset r*lh.
  std::int64_t off = 0;
  for (const AttentionInterior& in : parts) {
    const std::int64_t n = in.softmax_out.numel();
    std::memcpy(out + off, in.softmax_out.data(), sizeof(double) * static_cast<std::size_t>(n));
    std::memcpy(out + full + off, in.dropout_mask.data(), sizeof(double) * static_cast<std::size_t>(n));
    std::memcpy(out + 2 * full + off, in.dropout_out.data(), sizeof(double) * static_cast<std::size_t>(n));
    off += n;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// LayerParams::random(cfg, seed) (block.cpp:234-265), packed.
int ref_params_random(std::int64_t h, std::uint64_t seed, double* packed) {
  return guarded([&] {
    BlockConfig cfg;
    cfg.hidden = h;
    cfg.heads = 1;
    LayerParams p = LayerParams::random(cfg, seed);
    params_to(p, packed);
  });
}

// random_uniform(key, {n}, lo, hi) (rng.cpp:59-66).
void ref_random_uniform2(std::uint64_t key, std::int64_t n, double lo, double hi, double* out) {
  to_ptr(random_uniform(key, {n}, lo, hi), out);
}

std::uint64_t ref_hash_counter2(std::uint64_t key, std::uint64_t index) {
  return hash_counter(key, index);
}

// seqpar_block_forward (block.cpp:512-602) + seqpar_block_backward (block.cpp:622-749) on
// split(x, 0, t) / split(dy, 0, t). x, dy, y, dx are full {s,b,h}; grads are the assembled
// param_grads (block.cpp:730-746); w1_grad_shards {t, h, 4h/t}; interior {3, a, b, s, s};
// ledgers[t]. dy == NULL runs the forward only. Any output pointer may be NULL.
int ref_seqpar_layer(const CfgC* c, std::int64_t t, const double* params, const double* x,
                     const double* dy, double* y, double* dx, double* grads,
                     double* w1_grad_shards, double* interior, CommLogC* fwd_log,
                     CommLogC* bwd_log, LedgerC* ledgers) {
  return guarded([&] {
    const BlockConfig cfg = to_cfg(*c);
    const LayerParams p = params_from(cfg, params);
    const Tensor xf = from_ptr(x, {cfg.seq, cfg.batch, cfg.hidden});
    const SeqparForward fwd = seqpar_block_forward(split(xf, 0, t), p, t, cfg);
    if (y != nullptr) to_ptr(concat(fwd.y_shards, 0), y);
    if (interior != nullptr) {
      put_interior(fwd.interior, interior, cfg.heads * cfg.batch * cfg.seq * cfg.seq);
    }
    put_log(fwd.comm, fwd_log);
    if (ledgers != nullptr) {
      for (std::int64_t r = 0; r < t; ++r) put_ledger(fwd.ledgers[static_cast<std::size_t>(r)], &ledgers[r]);
    }
    if (dy == nullptr) return;
    const Tensor dyf = from_ptr(dy, {cfg.seq, cfg.batch, cfg.hidden});
    SeqparBackward back = seqpar_block_backward(split(dyf, 0, t), fwd, p);
    if (dx != nullptr) to_ptr(concat(back.dx_shards, 0), dx);
    if (grads != nullptr) params_to(back.param_grads, grads);
    if (w1_grad_shards != nullptr) {
      std::int64_t off = 0;
      for (const Tensor& g : back.w1_grad_shards) {
        to_ptr(g, w1_grad_shards + off);
        off += g.numel();
      }
    }
    put_log(back.comm, bwd_log);
  });
}

// reference_block_forward / reference_block_backward (block.cpp:419-510).
int ref_reference_layer(const CfgC* c, const double* params, const double* x, const double* dy,
                        double* y, double* dx, double* grads, double* q_out, double* k_out,
                        double* interior, LedgerC* ledger) {
  return guarded([&] {
    const BlockConfig cfg = to_cfg(*c);
    const LayerParams p = params_from(cfg, params);
    const ReferenceForward fwd =
        reference_block_forward(from_ptr(x, {cfg.seq, cfg.batch, cfg.hidden}), p, cfg);
    if (y != nullptr) to_ptr(fwd.y, y);
    if (q_out != nullptr) to_ptr(fwd.q, q_out);
    if (k_out != nullptr) to_ptr(fwd.k, k_out);
    if (interior != nullptr) {
      put_interior({fwd.interior}, interior, cfg.heads * cfg.batch * cfg.seq * cfg.seq);
    }
    put_ledger(fwd.ledger, ledger);
    if (dy == nullptr) return;
    BlockGrads g = reference_block_backward(from_ptr(dy, {cfg.seq, cfg.batch, cfg.hidden}), fwd, p);
    if (dx != nullptr) to_ptr(g.dx, dx);
    if (grads != nullptr) params_to(g.params, grads);
  });
}

// attention_interior(q, k, cfg, head_offset, local_heads) (block.cpp:381-417).
// q, k: {s, b, local_heads*hd}; outputs {local_heads, b, s, s} each.
int ref_attention_interior(const CfgC* c, const double* q, const double* k,
                           std::int64_t head_offset, std::int64_t local_heads,
                           double* softmax_out, double* dropout_mask, double* dropout_out) {
  return guarded([&] {
    const BlockConfig cfg = to_cfg(*c);
    const std::int64_t lw = local_heads * cfg.head_dim();
    const AttentionInterior in =
        attention_interior(from_ptr(q, {cfg.seq, cfg.batch, lw}), from_ptr(k, {cfg.seq, cfg.batch, lw}),
                           cfg, head_offset, local_heads);
    to_ptr(in.softmax_out, softmax_out);
    to_ptr(in.dropout_mask, dropout_mask);
    to_ptr(in.dropout_out, dropout_out);
  });
}

// all_gather / reduce_scatter / all_reduce over t equally-shaped shards (collectives.cpp:40-73).
// shards: t contiguous tensors of `shape` (ndim dims); log (optional) takes the counters
// under tag 0 schedule / 1 regather / 2 grad_sync.
int ref_all_gather(const double* shards, std::int64_t t, const std::int64_t* shape, std::int64_t ndim,
                   std::int64_t axis, double* out, CommLogC* log, int tag) {
  return guarded([&] {
    std::vector<std::int64_t> shp(shape, shape + ndim);
    std::vector<Tensor> parts;
    std::int64_t n = 1;
    for (auto d : shp) n *= d;
    for (std::int64_t r = 0; r < t; ++r) parts.push_back(from_ptr(shards + r * n, shp));
    CommLog cl;
    to_ptr(all_gather(parts, static_cast<std::size_t>(axis), &cl, static_cast<CommTag>(tag)), out);
    put_log(cl, log);
  });
}

int ref_reduce_scatter(const double* partials, std::int64_t t, const std::int64_t* shape,
                       std::int64_t ndim, std::int64_t axis, double* out, CommLogC* log, int tag) {
  return guarded([&] {
    std::vector<std::int64_t> shp(shape, shape + ndim);
    std::vector<Tensor> parts;
    std::int64_t n = 1;
    for (auto d : shp) n *= d;
    for (std::int64_t r = 0; r < t; ++r) parts.push_back(from_ptr(partials + r * n, shp));
    CommLog cl;
    std::vector<Tensor> res = reduce_scatter(parts, static_cast<std::size_t>(axis), &cl, static_cast<CommTag>(tag));
    std::int64_t off = 0;
    for (const Tensor& s : res) {
      to_ptr(s, out + off);
      off += s.numel();
    }
    put_log(cl, log);
  });
}

int ref_all_reduce(const double* partials, std::int64_t t, const std::int64_t* shape,
                   std::int64_t ndim, double* out, CommLogC* log, int tag) {
  return guarded([&] {
    std::vector<std::int64_t> shp(shape, shape + ndim);
    std::vector<Tensor> parts;
    std::int64_t n = 1;
    for (auto d : shp) n *= d;
    for (std::int64_t r = 0; r < t; ++r) parts.push_back(from_ptr(partials + r * n, shp));
    CommLog cl;
    to_ptr(all_reduce(parts, &cl, static_cast<CommTag>(tag)), out);
    put_log(cl, log);
  });
}

// layer_comm_bytes_tensor_parallel / _sequence (collectives.cpp:75-87).
std::int64_t ref_layer_comm_bytes_tp(std::int64_t s, std::int64_t b, std::int64_t h, std::int64_t t,
                                     std::int64_t e) {
  return actplan::to_int64(layer_comm_bytes_tensor_parallel(s, b, h, t, e));
}
std::int64_t ref_layer_comm_bytes_sp(std::int64_t s, std::int64_t b, std::int64_t h, std::int64_t t,
                                     std::int64_t e) {
  return actplan::to_int64(layer_comm_bytes_tensor_sequence(s, b, h, t, e));
}

}  // extern "C"
