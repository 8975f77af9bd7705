// The reference's own seqpar unit tests (/root/reference/proj/tests/test_seqpar.cpp:120-298),
// restated against the C++ facade (include/spl_seqpar.hpp) so they run on the B200 layer.
// Only the namespace and the GPU tolerances change (fp32 device arithmetic instead of fp64:
// 1e-5 where the reference asserts 1e-10 between t=1 and t=2).
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>

#include "spl_seqpar.hpp"

namespace seqpar = spl::seqpar;
using seqpar::BlockConfig;
using seqpar::LayerParams;
using seqpar::Tensor;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)
template <typename E>
static void check_throws(std::function<void()> f, const char* what) {
  ++g_checks;
  try {
    f();
  } catch (const E&) {
    return;
  } catch (...) {
  }
  ++g_fail;
  std::printf("FAIL: expected exception: %s\n", what);
}

static BlockConfig toy() {  // test_seqpar.cpp:31-39
  BlockConfig c;
  c.heads = 2; c.hidden = 8; c.seq = 4; c.batch = 1; c.seed = 7;
  return c;
}
static std::vector<Tensor> split0(const Tensor& x, int64_t t) {
  std::vector<Tensor> out;
  const int64_t rows = x.dim(0) / t, inner = x.numel() / x.dim(0);
  for (int64_t r = 0; r < t; ++r) {
    Tensor s({rows, x.dim(1), x.dim(2)});
    for (int64_t i = 0; i < rows * inner; ++i) s[i] = x[r * rows * inner + i];
    out.push_back(std::move(s));
  }
  return out;
}
static Tensor concat0(const std::vector<Tensor>& v) {
  int64_t rows = 0;
  for (auto& s : v) rows += s.dim(0);
  Tensor out({rows, v[0].dim(1), v[0].dim(2)});
  int64_t off = 0;
  for (auto& s : v) {
    for (int64_t i = 0; i < s.numel(); ++i) out[off + i] = s[i];
    off += s.numel();
  }
  return out;
}
using seqpar::max_abs_diff;
static Tensor tensor_of(std::vector<int64_t> shape, std::initializer_list<double> values) {
  Tensor out(std::move(shape));
  int64_t i = 0;
  for (double v : values) out[i++] = v;
  return out;
}
static int64_t group_bytes(const seqpar::ActivationLedger& l, std::initializer_list<const char*> names) {
  int64_t t = 0;
  for (auto& e : l.entries)
    for (auto* n : names)
      if (e.name == n) t += e.bytes;
  return t;
}

int main() {
  {  // reduce-scatter sums rank partials then shards them (test_seqpar.cpp:61-69)
    std::vector<Tensor> partials{tensor_of({2}, {1, 2}), tensor_of({2}, {3, 4})};
    const auto shards = seqpar::reduce_scatter(partials, 0);
    CHECK(shards.size() == 2 && shards[0][0] == 4 && shards[1][0] == 6);
  }
  {  // at t=1 every collective is the identity (71-79)
    std::vector<Tensor> one{tensor_of({2, 2}, {1, 2, 3, 4})};
    CHECK(seqpar::bit_equal(seqpar::all_gather(one, 0), one[0]));
    CHECK(seqpar::bit_equal(seqpar::all_reduce(one), one[0]));
    const auto sc = seqpar::reduce_scatter(one, 0);
    CHECK(sc.size() == 1 && seqpar::bit_equal(sc[0], one[0]));
  }
  {  // all_reduce equals all_gather of reduce_scatter on integer tensors (81-97)
    for (uint64_t trial = 0; trial < 50; ++trial) {
      std::vector<Tensor> partials;
      for (int64_t r = 0; r < 4; ++r) {
        Tensor part({8, 3});
        for (int64_t i = 0; i < part.numel(); ++i)
          part[i] = std::floor(seqpar::uniform01(seqpar::hash_counter(trial, (uint64_t)r), (uint64_t)i) * 33.0) - 16.0;
        partials.push_back(std::move(part));
      }
      CHECK(seqpar::bit_equal(seqpar::all_reduce(partials),
                              seqpar::all_gather(seqpar::reduce_scatter(partials, 0), 0)));
    }
    // CommLog ring model (collectives.cpp:30-38) and tags
    std::vector<Tensor> parts(4, Tensor({8, 3}));
    seqpar::CommLog log;
    seqpar::all_gather(parts, 1, &log, seqpar::CommTag::Regather);
    seqpar::reduce_scatter(parts, 0, &log);
    seqpar::all_reduce(parts, &log, seqpar::CommTag::GradSync);
    CHECK(log.regather.all_gathers == 1 && log.regather.ring_elements == (96 / 4) * 3);
    CHECK(log.schedule.reduce_scatters == 1 && log.schedule.ring_elements == (24 / 4) * 3);
    CHECK(log.grad_sync.all_reduces == 1 && log.grad_sync.ring_elements == 2 * (24 / 4) * 3);
    // axis 1 concatenation / scatter follow the reference's axis blocks (tensor.cpp:169-225)
    std::vector<Tensor> cols{tensor_of({2, 1}, {1, 2}), tensor_of({2, 1}, {3, 4})};
    CHECK(seqpar::bit_equal(seqpar::all_gather(cols, 1), tensor_of({2, 2}, {1, 3, 2, 4})));
    const auto rs = seqpar::reduce_scatter(std::vector<Tensor>{tensor_of({2, 2}, {1, 2, 3, 4}),
                                                               tensor_of({2, 2}, {10, 20, 30, 40})}, 1);
    CHECK(seqpar::bit_equal(rs[0], tensor_of({2, 1}, {11, 33})) &&
          seqpar::bit_equal(rs[1], tensor_of({2, 1}, {22, 44})));
  }
  {  // collectives reject ragged rank groups (99-107)
    std::vector<Tensor> ragged{Tensor({2, 2}), Tensor({2, 3})};
    check_throws<std::invalid_argument>([&] { seqpar::all_reduce(ragged); }, "ragged all_reduce");
    check_throws<std::invalid_argument>([&] { seqpar::all_gather(ragged, 0); }, "ragged all_gather");
    check_throws<std::invalid_argument>([&] { seqpar::reduce_scatter(ragged, 0); }, "ragged reduce_scatter");
    std::vector<Tensor> three(3, Tensor({4}));
    check_throws<std::invalid_argument>([&] { seqpar::reduce_scatter(three, 0); }, "indivisible scatter");
  }
  {  // sharded tensors reassemble and police their invariants (109-120)
    const Tensor full = seqpar::random_uniform(1, {4, 2, 6}, -1, 1);
    const auto sh = seqpar::RankShardedTensor::from_full(full, seqpar::ShardAxis::Sequence, 0, 2);
    CHECK(sh.shards.size() == 2);
    CHECK(seqpar::bit_equal(sh.to_full(0), full));
    sh.check();
    auto rep = seqpar::RankShardedTensor::from_full(full, seqpar::ShardAxis::Replicated, 0, 2);
    rep.check();
    rep.shards[1][0] += 1.0;
    check_throws<std::invalid_argument>([&] { rep.check(); }, "diverging replicas");
    // the RankShardedTensor overload of seqpar_block_forward (block.hpp:158-162)
    const BlockConfig cfg = toy();
    const LayerParams p = LayerParams::random(cfg, 31);
    const Tensor x = seqpar::random_uniform(32, {4, 1, 8}, -1, 1);
    auto a = seqpar::seqpar_block_forward(
        seqpar::RankShardedTensor::from_full(x, seqpar::ShardAxis::Sequence, 0, 2), p, cfg);
    auto b = seqpar::seqpar_block_forward(split0(x, 2), p, 2, cfg);
    CHECK(a.t == 2 && seqpar::bit_equal(concat0(a.y_shards), concat0(b.y_shards)));
    check_throws<std::invalid_argument>(
        [&] {
          seqpar::seqpar_block_forward(
              seqpar::RankShardedTensor::from_full(x, seqpar::ShardAxis::Hidden, 2, 2), p, cfg);
        },
        "hidden-sharded input");
  }
  {  // reference forward: ledger, zero block, p=0 masks, t=1 bit identity (122-168)
    BlockConfig cfg = toy();
    const LayerParams p = LayerParams::random(cfg, 11);
    const Tensor x = seqpar::random_uniform(3, {4, 1, 8}, -1, 1);
    const auto fwd = seqpar::reference_block_forward(x, p, cfg);
    CHECK(fwd.ledger.total_bytes() == 1248);
    CHECK(fwd.ledger.total_bytes() == seqpar::layer_component_breakdown(2, 8, 4, 1).total);
    const auto z = seqpar::reference_block_forward(Tensor({4, 1, 8}), LayerParams::zeros(cfg), cfg);
    bool zero = true;
    for (int64_t i = 0; i < z.y.numel(); ++i) zero &= z.y[i] == 0.0;
    CHECK(zero);
    cfg.dropout_p = 0.0;
    const LayerParams p5 = LayerParams::random(cfg, 5);
    const Tensor x9 = seqpar::random_uniform(9, {4, 1, 8}, -1, 1);
    const auto dry = seqpar::reference_block_forward(x9, p5, cfg);
    const Tensor m = dry.attn_dropout_mask();
    bool ones = m.numel() == 32;
    for (int64_t i = 0; i < m.numel(); ++i) ones &= m[i] == 1.0;
    CHECK(ones);
    cfg.dropout_p = 0.25;
    CHECK(seqpar::reference_block_forward(x9, p5, cfg).ledger.total_bytes() == dry.ledger.total_bytes());
    const BlockConfig c0 = toy();
    const LayerParams p21 = LayerParams::random(c0, 21);
    const Tensor x22 = seqpar::random_uniform(22, {4, 1, 8}, -1, 1);
    CHECK(seqpar::bit_equal(seqpar::seqpar_block_forward({x22}, p21, 1, c0).y_shards[0],
                            seqpar::reference_block_forward(x22, p21, c0).y));
    // reference backward == seqpar t=1 backward
    const Tensor dy = seqpar::random_uniform(23, {4, 1, 8}, -1, 1);
    const auto rf = seqpar::reference_block_forward(x22, p21, c0);
    const auto rg = seqpar::reference_block_backward(dy, rf, p21);
    const auto sf = seqpar::seqpar_block_forward({x22}, p21, 1, c0);
    const auto sg = seqpar::seqpar_block_backward({dy}, sf, p21);
    CHECK(seqpar::bit_equal(rg.dx, sg.dx_shards[0]));
    CHECK(seqpar::bit_equal(rg.params.w1, sg.param_grads.w1));
    check_throws<std::invalid_argument>([&] { seqpar::reference_block_forward(Tensor({2, 1, 8}), p21, c0); },
                                        "reference input shape");
    // backward with other params: the GEMMs use them (block.cpp:639-640)
    const LayerParams other = LayerParams::random(c0, 99);
    const auto og = seqpar::reference_block_backward(dy, seqpar::reference_block_forward(x22, p21, c0), other);
    CHECK(!seqpar::bit_equal(og.dx, rg.dx));
  }
  {  // attention_interior(q, k, cfg, head_offset, local_heads) (block.cpp:381-417)
    BlockConfig cfg;
    cfg.heads = 4; cfg.hidden = 32; cfg.seq = 16; cfg.batch = 2; cfg.dropout_p = 0.1; cfg.causal = true;
    const Tensor q = seqpar::random_uniform(41, {16, 2, 32}, -1, 1);
    const Tensor k = seqpar::random_uniform(42, {16, 2, 32}, -1, 1);
    const auto full = seqpar::attention_interior(q, k, cfg, 0, 4);
    // head slice 2..3 = the rank-1 view at t=2: columns 16..31 of q/k
    Tensor q1({16, 2, 16}), k1({16, 2, 16});
    for (int64_t r = 0; r < 32; ++r)
      for (int64_t c = 0; c < 16; ++c) {
        q1[r * 16 + c] = q[r * 32 + 16 + c];
        k1[r * 16 + c] = k[r * 32 + 16 + c];
      }
    const auto half = seqpar::attention_interior(q1, k1, cfg, 2, 2);
    const int64_t per = 2 * 2 * 16 * 16;
    bool same_mask = true, same_sm = true, rows_ok = true, drop_ok = true;
    for (int64_t i = 0; i < per; ++i) {
      same_mask &= half.dropout_mask[i] == full.dropout_mask[per + i];
      same_sm &= std::abs(half.softmax_out[i] - full.softmax_out[per + i]) <= 1e-6;
      drop_ok &= std::abs(half.dropout_out[i] - half.softmax_out[i] * half.dropout_mask[i] / 0.9) <= 1e-6;
    }
    for (int64_t row = 0; row < 2 * 2 * 16; ++row) {
      double sum = 0;
      for (int64_t j = 0; j < 16; ++j) {
        sum += half.softmax_out[row * 16 + j];
        if (j > row % 16) rows_ok &= half.softmax_out[row * 16 + j] == 0.0;  // causal
      }
      rows_ok &= std::abs(sum - 1.0) <= 1e-5;
    }
    CHECK(same_mask && same_sm && rows_ok && drop_ok);
    check_throws<std::invalid_argument>([&] { seqpar::attention_interior(q1, k1, cfg, 1, 2); },
                                        "misaligned head offset");
  }
  {  // RecomputeStrategy::parse / name (test_config.cpp:92-106)
    using S = seqpar::RecomputeStrategy;
    for (const char* n : {"none", "full", "selective", "none+seq", "full+seq", "selective+seq",
                          "full+mblevel", "selective+seq+mblevel"})
      CHECK(S::parse(n).name() == n);
    CHECK(S::parse("full+seq").sequence_parallel);
    CHECK(S::parse("selective+mblevel").microbatch_level);
    CHECK(S::parse("seq+selective") == S::parse("selective+seq"));
    for (const char* bad : {"none+mblevel", "bogus", "full+bogus", "full+selective", "seq"})
      check_throws<std::invalid_argument>([&] { S::parse(bad); }, bad);
  }
  {  // ledger matches the itemised toy count (test_seqpar.cpp:120-137)
    const BlockConfig cfg = toy();
    const LayerParams p = LayerParams::random(cfg, 11);
    const Tensor x = seqpar::random_uniform(3, {4, 1, 8}, -1, 1);
    auto f = seqpar::seqpar_block_forward({x}, p, 1, cfg);
    CHECK(f.ledgers[0].total_bytes() == 1248);
    CHECK(group_bytes(f.ledgers[0], {"qkv_input", "query", "key", "value", "softmax_out",
                                     "softmax_dropout_mask", "softmax_dropout_out",
                                     "attn_proj_input", "attn_dropout_mask"}) == 512);
    CHECK(group_bytes(f.ledgers[0], {"mlp_fc1_input", "gelu_input", "mlp_fc2_input", "mlp_dropout_mask"}) == 608);
    CHECK(group_bytes(f.ledgers[0], {"ln1_input", "ln2_input"}) == 128);
  }
  {  // zero input and zero weights flow to a zero output (139-145)
    const BlockConfig cfg = toy();
    auto f = seqpar::seqpar_block_forward({Tensor({4, 1, 8})}, LayerParams::zeros(cfg), 1, cfg);
    bool zero = true;
    for (int64_t i = 0; i < f.y_shards[0].numel(); ++i) zero &= f.y_shards[0][i] == 0.0;
    CHECK(zero);
  }
  {  // t=2 matches t=1 and each rank stores half the footprint (161-183)
    BlockConfig cfg = toy();
    const LayerParams p = LayerParams::random(cfg, 31);
    const Tensor x = seqpar::random_uniform(32, {4, 1, 8}, -1, 1);
    auto f1 = seqpar::seqpar_block_forward({x}, p, 1, cfg);
    auto f2 = seqpar::seqpar_block_forward(split0(x, 2), p, 2, cfg);
    CHECK(max_abs_diff(concat0(f2.y_shards), f1.y_shards[0]) <= 1e-5);
    for (auto& l : f2.ledgers) CHECK(l.total_bytes() * 2 == f1.ledgers[0].total_bytes());
    cfg.causal = true;  // 185-199
    auto c1 = seqpar::seqpar_block_forward({x}, p, 1, cfg);
    auto c2 = seqpar::seqpar_block_forward(split0(x, 2), p, 2, cfg);
    CHECK(max_abs_diff(concat0(c2.y_shards), c1.y_shards[0]) <= 1e-5);
  }
  {  // backward matches and sharded grads stay local (201-232)
    BlockConfig cfg = toy();
    cfg.heads = 4;
    const LayerParams p = LayerParams::random(cfg, 51);
    const Tensor x = seqpar::random_uniform(52, {4, 1, 8}, -1, 1);
    const Tensor dy = seqpar::random_uniform(53, {4, 1, 8}, -1, 1);
    auto f1 = seqpar::seqpar_block_forward({x}, p, 1, cfg);
    auto b1 = seqpar::seqpar_block_backward({dy}, f1, p);
    auto f2 = seqpar::seqpar_block_forward(split0(x, 2), p, 2, cfg);
    auto b2 = seqpar::seqpar_block_backward(split0(dy, 2), f2, p);
    CHECK(max_abs_diff(concat0(b2.dx_shards), b1.dx_shards[0]) <= 1e-4);
    auto g1 = b1.param_grads.all();
    auto g2 = b2.param_grads.all();
    for (size_t i = 0; i < g1.size(); ++i) CHECK(max_abs_diff(*g2[i], *g1[i]) <= 1e-4);
    for (int r = 0; r < 2; ++r) {
      const Tensor& s = b2.w1_grad_shards[(size_t)r];
      double m = 0;
      for (int64_t i = 0; i < 8; ++i)
        for (int64_t j = 0; j < 16; ++j)
          m = std::max(m, std::abs(s[i * 16 + j] - b1.param_grads.w1[i * 32 + r * 16 + j]));
      CHECK(m <= 1e-4);
    }
    CHECK(b2.comm.schedule.all_gathers == 2 && b2.comm.schedule.reduce_scatters == 2);
    CHECK(f2.comm.schedule.all_gathers == 2 && f2.comm.schedule.reduce_scatters == 2);
    CHECK(b2.comm.regather.all_gathers == 2 && b2.comm.grad_sync.all_reduces == 6);
  }
  {  // an identity-like block passes gradients through exactly (234-246)
    const BlockConfig cfg = toy();
    const LayerParams p = LayerParams::zeros(cfg);
    const Tensor dy = seqpar::random_uniform(61, {4, 1, 8}, -1, 1);
    auto f = seqpar::seqpar_block_forward({Tensor({4, 1, 8})}, p, 1, cfg);
    auto b = seqpar::seqpar_block_backward({dy}, f, p);
    double m = 0;
    for (int64_t i = 0; i < dy.numel(); ++i) m = std::max(m, std::abs(b.dx_shards[0][i] - (double)(float)dy[i]));
    CHECK(m == 0.0);
  }
  {  // shard mismatches and missing state raise errors (273-298)
    const BlockConfig cfg = toy();
    const LayerParams p = LayerParams::random(cfg, 81);
    const Tensor x = seqpar::random_uniform(82, {4, 1, 8}, -1, 1);
    check_throws<std::invalid_argument>([&] { seqpar::seqpar_block_forward(split0(x, 2), p, 4, cfg); },
                                        "t mismatch");
    auto f = seqpar::seqpar_block_forward(split0(x, 2), p, 2, cfg);
    check_throws<std::invalid_argument>(
        [&] { seqpar::seqpar_block_backward({Tensor({1, 1, 8}), Tensor({1, 1, 8})}, f, p); },
        "dy shape");
    seqpar::SeqparForward empty;
    empty.t = 2;
    empty.cfg = cfg;
    check_throws<std::invalid_argument>([&] { seqpar::seqpar_block_backward(split0(x, 2), empty, p); },
                                        "missing state");
    Tensor bad({4, 1, 8});
    bad[0] = std::numeric_limits<double>::infinity();
    check_throws<std::domain_error>([&] { seqpar::seqpar_block_forward({bad}, p, 1, cfg); }, "non-finite");
  }
  {  // accountant pins (test_activation_memory.cpp:42-57)
    using K = seqpar::RecomputeKind;
    CHECK(seqpar::per_layer_bytes(64, 6144, 2048, 4, 1, K::None, false) == 7079985152LL);
    CHECK(seqpar::per_layer_bytes(64, 6144, 2048, 4, 8, K::None, true) == 884998144LL);
    CHECK(seqpar::per_layer_bytes(64, 6144, 2048, 4, 8, K::Selective, true) == 213909504LL);
    // test_activation_memory.cpp:59-66, 97-99, 198-206; collectives.cpp:75-87
    const auto bd = seqpar::layer_component_breakdown(2, 8, 4, 1);
    CHECK(bd.attention == 512 && bd.mlp == 608 && bd.layer_norms == 128 && bd.total == 1248);
    const auto pb = seqpar::percent_of_baseline(128, 20480, 2048, 1, 8, K::Selective, true);
    CHECK(pb.num == 17 && pb.den == 84);
    CHECK(seqpar::total_first_stage_bytes(128, 20480, 2048, 1, 8, K::Selective, true, 105, 35, 3) ==
          24777850880LL);
    CHECK(seqpar::layer_comm_bytes_tensor_sequence(2048, 4, 6144, 8, 2) ==
          seqpar::layer_comm_bytes_tensor_parallel(2048, 4, 6144, 8, 2));
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
