// The reference's microbatch-window cases (/root/reference/proj/tests/test_pipeline_sim.cpp,
// "window plan reproduces the moving-window scenario", "window plan boundary budgets",
// "in-flight bound") restated against the C++ facade (include/spl_pipeline.hpp) — host-only,
// no GPU needed. Expected values are the reference's own.
#include <cstdio>
#include <functional>
#include <limits>

#include "spl_pipeline.hpp"

namespace pipeline = spl::pipeline;
using pipeline::ParallelLayout;
using pipeline::RecomputeKind;
using pipeline::RecomputeStrategy;
using pipeline::StoredMode;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    ++g_checks;                                                   \
    if (!(cond)) {                                                \
      ++g_fail;                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                             \
  } while (0)

static const pipeline::ModelShape kToy{2, 8, 8, 4, 16};  // a, h, L, s, v

static ParallelLayout layout_of(int64_t p, int64_t n_mb) {
  ParallelLayout l;
  l.pipeline = p;
  l.microbatches_per_iter = n_mb;
  return l;
}
static RecomputeStrategy kind_of(RecomputeKind k) {
  RecomputeStrategy s;
  s.kind = k;
  return s;
}
static int64_t per_layer(RecomputeKind k) {
  int64_t v = 0;
  spl_per_layer_bytes(kToy.attention_heads, kToy.hidden, kToy.seq_len, 1, 1, (int)k, 0, 2, 1, &v);
  return v;
}

int main() {
  const int64_t kMax = std::numeric_limits<int64_t>::max();
  // in_flight (test_pipeline_sim.cpp, "in-flight bound is max(0, p - S)")
  CHECK(pipeline::in_flight(35, 0) == 35);
  CHECK(pipeline::in_flight(4, 3) == 1);
  CHECK(pipeline::in_flight(4, 7) == 0);

  {  // moving-window scenario at p = 4, n_mb = 9, inner = full
    const ParallelLayout layout = layout_of(4, 9);
    const RecomputeStrategy inner = kind_of(RecomputeKind::Full);
    const int64_t lps = kToy.layers / layout.pipeline;
    const int64_t extras = kToy.seq_len * kToy.hidden;  // embedding-dropout mask, 1 B, t = 1
    const int64_t full_mb = per_layer(RecomputeKind::None) * lps + extras;
    const int64_t ckpt_mb = per_layer(RecomputeKind::Full) * lps + extras;
    const pipeline::WindowPlan plan =
        pipeline::microbatch_window_plan(kToy, layout, inner, full_mb + 3 * ckpt_mb);
    std::vector<int> stored;
    for (int mb = 1; mb <= 9; ++mb)
      if (plan.modes[0][(size_t)mb - 1] == StoredMode::FullyStored) stored.push_back(mb);
    CHECK((stored == std::vector<int>{1, 5, 9}));
    CHECK(plan.per_stage[0].fully_stored == 3 && plan.per_stage[0].checkpointed == 6);
    for (size_t s = 1; s < plan.per_stage.size(); ++s)
      CHECK(plan.per_stage[s].checkpointed <= plan.per_stage[s - 1].checkpointed);
    CHECK(plan.per_stage.back().checkpointed == 0);
    CHECK((plan.recomputed_fraction == pipeline::Rational{4, 9}));  // (6+6+4+0)/36
  }
  {  // boundary budgets, inner = selective
    const ParallelLayout layout = layout_of(4, 9);
    const RecomputeStrategy inner = kind_of(RecomputeKind::Selective);
    const pipeline::WindowPlan all = pipeline::microbatch_window_plan(kToy, layout, inner, kMax);
    for (const auto& st : all.per_stage) CHECK(st.checkpointed == 0);
    CHECK((all.recomputed_fraction == pipeline::Rational{0, 1}));
    const pipeline::WindowPlan tight =
        pipeline::microbatch_window_plan(kToy, layout, inner, all.min_feasible_budget);
    CHECK(tight.per_stage[0].fully_stored == 0 && tight.per_stage[0].checkpointed == 9);
    const ParallelLayout single = layout_of(1, 3);
    const pipeline::WindowPlan probe = pipeline::microbatch_window_plan(kToy, single, inner, kMax);
    const pipeline::WindowPlan one =
        pipeline::microbatch_window_plan(kToy, single, inner, probe.min_feasible_budget);
    CHECK(one.per_stage[0].fully_stored == 0);
    CHECK((one.recomputed_fraction == pipeline::Rational{1, 1}));
    bool thrown = false;
    try {
      pipeline::microbatch_window_plan(kToy, layout, inner, 16);
    } catch (const pipeline::InfeasibleBudgetError& e) {
      thrown = true;
      CHECK(e.min_feasible_budget > 16);
      const pipeline::WindowPlan ok =
          pipeline::microbatch_window_plan(kToy, layout, inner, e.min_feasible_budget);
      CHECK(ok.min_feasible_budget == e.min_feasible_budget);
    }
    CHECK(thrown);
  }
  {  // invalid configurations: n_mb < p, inner none
    bool a = false, b = false;
    try {
      pipeline::microbatch_window_plan(kToy, layout_of(4, 3), kind_of(RecomputeKind::Full), kMax);
    } catch (const std::invalid_argument&) {
      a = true;
    }
    try {
      pipeline::microbatch_window_plan(kToy, layout_of(2, 4), kind_of(RecomputeKind::None), kMax);
    } catch (const std::invalid_argument&) {
      b = true;
    }
    CHECK(a && b);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
