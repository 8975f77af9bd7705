// Microbatch-level recompute window: planner (exact integer arithmetic, host) — see window.hpp.
#include <algorithm>
#include <string>

#include "common.hpp"
#include "layer.hpp"
#include "window.hpp"

namespace spl {

std::vector<ProgEvent> rank_program(int64_t p, int64_t stage, int64_t n_mb) {
  // p-S warm-up forwards, then backward/forward alternation, then the backward drain
  // (pipeline_sim.cpp:40-56)
  std::vector<ProgEvent> prog;
  const int64_t warmup = p - stage;
  int64_t fwd = 0, bwd = 0;
  for (; fwd < warmup; ++fwd) prog.push_back({true, (int32_t)(fwd + 1)});
  while (bwd < n_mb) {
    ++bwd;
    prog.push_back({false, (int32_t)bwd});
    if (fwd < n_mb) {
      ++fwd;
      prog.push_back({true, (int32_t)fwd});
    }
  }
  return prog;
}

void validate_model(const spl_model_desc& m) {
  std::string what;
  auto need = [&](bool ok, const char* field, const char* msg) {
    if (!ok) what += std::string(" [") + field + "] " + msg + ";";
  };
  need(m.heads >= 1, "a", "a must be >= 1");
  need(m.hidden >= 1, "h", "h must be >= 1");
  need(m.layers >= 1, "L", "L must be >= 1");
  need(m.seq >= 1, "s", "s must be >= 1");
  need(m.vocab >= 1, "v", "v must be >= 1");
  need(m.tensor >= 1, "t", "t must be >= 1");
  need(m.pipeline >= 1, "p", "p must be >= 1");
  need(m.interleave >= 1, "m", "m must be >= 1");
  need(m.microbatch >= 1, "b", "b must be >= 1");
  need(m.microbatches >= 1, "n_mb", "n_mb must be >= 1");
  if (m.heads >= 1 && m.hidden >= 1)
    need(m.hidden % m.heads == 0, "h", "h not divisible by a (head dim must be integral)");
  if (m.hidden >= 1 && m.tensor >= 1) need(m.hidden % m.tensor == 0, "h", "h not divisible by t");
  if (m.seq >= 1 && m.tensor >= 1) need(m.seq % m.tensor == 0, "s", "s not divisible by t");
  if (m.layers >= 1 && m.pipeline >= 1 && m.interleave >= 1)
    need(m.layers % (m.pipeline * m.interleave) == 0, "L", "L not divisible by p*m");
  if (m.pipeline >= 1 && m.microbatches >= 1)
    need(m.microbatches >= m.pipeline, "n_mb", "n_mb < p (pipeline cannot be filled)");
  if (!what.empty()) raise(SPL_EINVAL, "invalid configuration:" + what);
  require(m.act_bytes >= 1 && m.mask_bytes >= 1 && m.logits_bytes >= 1,
          "byte convention widths must be >= 1");
  require(m.recompute >= 0 && m.recompute <= 2, "unknown recompute kind");
}

namespace {
int64_t fit(__int128 v) {
  if (v > (__int128)INT64_MAX || v < (__int128)INT64_MIN)
    raise(SPL_EINVAL, "value does not fit in 64-bit integer");
  return (int64_t)v;
}
// floor(per_layer(kind) · L/p + extras), extras = en / t (activation_memory.cpp:125-137)
int64_t stage_bytes(const spl_model_desc& m, int kind, __int128 extras_num) {
  __int128 n, d;
  if (per_layer_bytes_exact(m.heads, m.hidden, m.seq, m.microbatch, m.tensor, kind,
                            m.sequence_parallel, m.act_bytes, m.mask_bytes, &n, &d))
    raise(SPL_EINVAL, "invalid configuration");
  const __int128 lps = m.layers / m.pipeline;
  const __int128 t = m.tensor;
  return fit((n * lps * t + extras_num * d) / (d * t));
}
__int128 gcd(__int128 x, __int128 y) {
  while (y) {
    const __int128 r = x % y;
    x = y;
    y = r;
  }
  return x;
}
}  // namespace

MbBytes microbatch_bytes(const spl_model_desc& m, int64_t stage) {
  validate_model(m);
  require(stage >= 0 && stage < m.pipeline, "stage must lie in [0, p)");
  const __int128 sbh = (__int128)m.seq * m.microbatch * m.hidden;
  __int128 extras = 0;  // numerator over t
  if (stage == 0) {
    extras += (__int128)m.mask_bytes * sbh;  // embedding-dropout mask shard
    if (m.pipeline == 1)                     // output side: 2 activations + the logits
      extras += (__int128)2 * m.act_bytes * sbh +
                (__int128)m.logits_bytes * m.seq * m.microbatch * m.vocab;
  }
  MbBytes out;
  out.fully_stored = stage_bytes(m, SPL_RECOMPUTE_NONE, extras);
  out.checkpointed =
      m.recompute == SPL_RECOMPUTE_NONE ? out.fully_stored : stage_bytes(m, m.recompute, extras);
  return out;
}

WindowPlanOut window_plan(const spl_model_desc& m, int64_t budget, int64_t* min_budget_out) {
  validate_model(m);
  if (m.recompute == SPL_RECOMPUTE_NONE)
    raise(SPL_EINVAL, "window plan needs a full or selective inner strategy");
  const int64_t p = m.pipeline, n_mb = m.microbatches;
  WindowPlanOut plan;
  plan.modes.assign((size_t)(p * n_mb), 0);
  plan.stage_counts.assign((size_t)(2 * p), 0);
  std::vector<MbBytes> sb;
  int64_t min_budget = 0;
  for (int64_t s = 0; s < p; ++s) {
    sb.push_back(microbatch_bytes(m, s));
    const __int128 need = (__int128)(p - s) * sb.back().checkpointed;
    min_budget = std::max<int64_t>(min_budget, fit(need));
  }
  plan.min_feasible_budget = min_budget;
  if (min_budget_out) *min_budget_out = min_budget;
  if (budget < min_budget)
    raise(SPL_EBUDGET, "budget " + std::to_string(budget) +
                           " bytes cannot hold the all-checkpointed schedule; minimum feasible "
                           "budget is " + std::to_string(min_budget) + " bytes");
  __int128 recomputed = 0;
  for (int64_t s = 0; s < p; ++s) {
    const MbBytes& mb = sb[(size_t)s];
    const int64_t slots = p - s;
    int64_t live_full = 0, n_full = 0, n_ckpt = 0;
    uint8_t* row = &plan.modes[(size_t)(s * n_mb)];
    for (const ProgEvent& ev : rank_program(p, s, n_mb)) {
      if (ev.forward) {
        // worst-case projected peak if this microbatch keeps everything: the live fully stored
        // ones plus it, the remaining in-flight slots refilled with checkpointed microbatches
        const __int128 projected = (__int128)(live_full + 1) * mb.fully_stored +
                                   (__int128)std::max<int64_t>(0, slots - (live_full + 1)) *
                                       mb.checkpointed;
        if (projected <= budget) {
          row[ev.microbatch - 1] = 1;
          ++live_full;
          ++n_full;
        } else {
          ++n_ckpt;
        }
      } else if (row[ev.microbatch - 1]) {
        --live_full;
      }
    }
    plan.stage_counts[(size_t)(2 * s)] = n_full;
    plan.stage_counts[(size_t)(2 * s + 1)] = n_ckpt;
    recomputed += n_ckpt;
  }
  const __int128 den = (__int128)p * n_mb, g = gcd(recomputed, den);
  plan.rec_num = g ? recomputed / g : 0;
  plan.rec_den = g ? den / g : 1;
  return plan;
}

int64_t stage_timeline(const spl_model_desc& m, int64_t stage, const uint8_t* modes_row,
                       bool dealloc, std::vector<int64_t>* bytes_after) {
  const MbBytes mb = microbatch_bytes(m, stage);  // validates
  require(modes_row != nullptr, "null modes row");
  const bool recompute = m.recompute != SPL_RECOMPUTE_NONE;
  const int64_t out_tensor = fit((__int128)m.act_bytes * m.seq * m.microbatch * m.hidden);
  __int128 cur = 0;
  int64_t peak = 0;
  for (const ProgEvent& ev : rank_program(m.pipeline, stage, m.microbatches)) {
    const bool full = modes_row[ev.microbatch - 1] != 0;
    const int64_t stored = full ? mb.fully_stored : mb.checkpointed;
    if (ev.forward) {
      cur += stored;
      if (!dealloc) cur += out_tensor;
    } else {
      if (recompute && !full && bytes_after) bytes_after->push_back(fit(cur));  // Recompute
      cur -= stored;
      if (!dealloc) cur -= out_tensor;
    }
    if (bytes_after) bytes_after->push_back(fit(cur));
    peak = std::max<int64_t>(peak, fit(cur));
  }
  return peak;
}

}  // namespace spl
