// spl_pipeline.hpp — header-only C++ facade over the C ABI (spl.h) for the microbatch-level
// recompute window, with the reference's signatures, so code written against actplan::pipeline
// (pipeline_sim.hpp) and actplan config types (config.hpp) switches by changing the namespace:
// `namespace pipeline = spl::pipeline;`.
//
//   reference (actplan)                                    facade (spl::pipeline)
//   ModelShape / ParallelLayout      config.hpp:27-48      ModelShape / ParallelLayout
//   RecomputeStrategy                config.hpp:53-70      RecomputeStrategy
//   ByteConvention                   config.hpp:74-80      ByteConvention
//   pipeline::in_flight              pipeline_sim.hpp:46   in_flight
//   pipeline::StoredMode, StageWindow, WindowPlan  :29-105 StoredMode, StageWindow, WindowPlan
//   pipeline::InfeasibleBudgetError  pipeline_sim.hpp:98   InfeasibleBudgetError
//   pipeline::microbatch_window_plan pipeline_sim.hpp:108  microbatch_window_plan
// Rational (Boost cpp_rational) becomes a reduced int64 num/den pair. Errors:
// std::invalid_argument where the reference throws it, InfeasibleBudgetError for a budget below
// the all-checkpointed schedule. The executor of a planned window on the GPU is spl_window_* in
// spl.h.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "spl.h"

namespace spl::pipeline {

struct ModelShape {
  int64_t attention_heads = 0, hidden = 0, layers = 0, seq_len = 0, vocab = 0;
};
struct ParallelLayout {
  int64_t tensor = 1, pipeline = 1, interleave = 1, data_parallel = 1, microbatch = 1,
          microbatches_per_iter = 1;
};
enum class RecomputeKind { None = SPL_RECOMPUTE_NONE, Full = SPL_RECOMPUTE_FULL,
                           Selective = SPL_RECOMPUTE_SELECTIVE };
struct RecomputeStrategy {
  RecomputeKind kind = RecomputeKind::None;
  bool sequence_parallel = false;
  bool microbatch_level = false;
};
struct ByteConvention {
  int64_t activation_elem = 2, mask_elem = 1, logits_elem = 4;
};

enum class StoredMode { Checkpointed, FullyStored };
using StoredModeAssignment = std::vector<std::vector<StoredMode>>;
struct StageWindow {
  int64_t fully_stored = 0, checkpointed = 0;
};
struct Rational {
  int64_t num = 0, den = 1;
  bool operator==(const Rational& o) const { return num == o.num && den == o.den; }
};
struct WindowPlan {
  std::vector<StageWindow> per_stage;
  StoredModeAssignment modes;  // modes[rank][mb - 1]
  Rational recomputed_fraction;
  int64_t min_feasible_budget = 0;
};

class InfeasibleBudgetError : public std::runtime_error {
 public:
  InfeasibleBudgetError(const std::string& what, int64_t min_budget)
      : std::runtime_error(what), min_feasible_budget(min_budget) {}
  int64_t min_feasible_budget;
};

inline int64_t in_flight(int64_t p, int64_t stage) {
  if (stage < 0) throw std::invalid_argument("stage must be >= 0");
  return p - stage > 0 ? p - stage : 0;
}

namespace detail {
inline spl_model_desc desc(const ModelShape& s, const ParallelLayout& l,
                           const RecomputeStrategy& r, const ByteConvention& c) {
  spl_model_desc m;
  spl_model_desc_default(&m);
  m.heads = s.attention_heads;
  m.hidden = s.hidden;
  m.layers = s.layers;
  m.seq = s.seq_len;
  m.vocab = s.vocab;
  m.tensor = l.tensor;
  m.pipeline = l.pipeline;
  m.interleave = l.interleave;
  m.microbatch = l.microbatch;
  m.microbatches = l.microbatches_per_iter;
  m.recompute = (int32_t)r.kind;
  m.sequence_parallel = r.sequence_parallel ? 1 : 0;
  m.act_bytes = c.activation_elem;
  m.mask_bytes = c.mask_elem;
  m.logits_bytes = c.logits_elem;
  return m;
}
}  // namespace detail

inline WindowPlan microbatch_window_plan(const ModelShape& shape, const ParallelLayout& layout,
                                         const RecomputeStrategy& inner, int64_t budget,
                                         const ByteConvention& conv = {}) {
  const spl_model_desc m = detail::desc(shape, layout, inner, conv);
  const int64_t p = layout.pipeline > 0 ? layout.pipeline : 0;
  const int64_t n = layout.microbatches_per_iter > 0 ? layout.microbatches_per_iter : 0;
  std::vector<uint8_t> modes((size_t)(p * n > 0 ? p * n : 1));
  std::vector<int64_t> counts((size_t)(2 * p > 0 ? 2 * p : 2));
  int64_t num = 0, den = 1, minb = 0;
  const int rc = spl_window_plan(&m, budget, modes.data(), counts.data(), &num, &den, &minb);
  if (rc == SPL_EBUDGET) throw InfeasibleBudgetError(spl_last_error(), minb);
  if (rc == SPL_EINVAL) throw std::invalid_argument(spl_last_error());
  if (rc != SPL_OK) throw std::runtime_error(spl_last_error());
  WindowPlan plan;
  plan.min_feasible_budget = minb;
  plan.recomputed_fraction = {num, den};
  for (int64_t s = 0; s < p; ++s) {
    plan.per_stage.push_back({counts[(size_t)(2 * s)], counts[(size_t)(2 * s + 1)]});
    std::vector<StoredMode> row;
    for (int64_t i = 0; i < n; ++i)
      row.push_back(modes[(size_t)(s * n + i)] ? StoredMode::FullyStored
                                               : StoredMode::Checkpointed);
    plan.modes.push_back(row);
  }
  return plan;
}

}  // namespace spl::pipeline
