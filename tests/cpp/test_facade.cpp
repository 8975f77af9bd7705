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
static double max_abs_diff(const Tensor& a, const Tensor& b) {
  double m = 0;
  for (int64_t i = 0; i < a.numel(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}
static int64_t group_bytes(const seqpar::ActivationLedger& l, std::initializer_list<const char*> names) {
  int64_t t = 0;
  for (auto& e : l.entries)
    for (auto* n : names)
      if (e.name == n) t += e.bytes;
  return t;
}

int main() {
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
