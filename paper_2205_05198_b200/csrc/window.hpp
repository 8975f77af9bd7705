// Microbatch-level recompute window: the planner of the reference's
// microbatch_window_plan / simulate_memory_with_modes restricted to one pipeline rank's program
// (pipeline_sim.cpp:26-56, 222-359), and the executor that runs that rank program on the GPU
// with real layer stacks: fully-stored microbatches on a no-recompute stack, checkpointed ones
// on a stack of the inner regime, parameters and gradients shared between them.
#pragma once
#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "../../include/spl.h"

namespace spl {

// One event of a rank's 1F1B program (pipeline_sim.cpp:40-56); microbatch is 1-based.
struct ProgEvent {
  bool forward;
  int32_t microbatch;
};
std::vector<ProgEvent> rank_program(int64_t p, int64_t stage, int64_t n_mb);

void validate_model(const spl_model_desc& m);  // config.cpp:86-133

struct MbBytes {
  int64_t fully_stored = 0, checkpointed = 0;
};
// microbatch_bytes (pipeline_sim.cpp:192-220): L/p layers of per-layer bytes plus the
// first-stage extras (and the output extras at p = 1), floored once.
MbBytes microbatch_bytes(const spl_model_desc& m, int64_t stage);

struct WindowPlanOut {
  std::vector<uint8_t> modes;         // [p][n_mb], 1 = fully stored
  std::vector<int64_t> stage_counts;  // [p][2]: fully stored, checkpointed
  __int128 rec_num = 0, rec_den = 1;  // recomputed fraction, reduced
  int64_t min_feasible_budget = 0;
};
// microbatch_window_plan (pipeline_sim.cpp:297-359). Throws Error(SPL_EBUDGET) with
// *min_budget_out set when the budget cannot hold the all-checkpointed schedule.
WindowPlanOut window_plan(const spl_model_desc& m, int64_t budget, int64_t* min_budget_out);

// Per-rank activation timeline of simulate_memory_with_modes (pipeline_sim.cpp:222-275): bytes
// after each program event of `stage` (recompute events hold the count), and the peak.
int64_t stage_timeline(const spl_model_desc& m, int64_t stage, const uint8_t* modes_row,
                       bool dealloc, std::vector<int64_t>* bytes_after);

}  // namespace spl
