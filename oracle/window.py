"""Microbatch-level recompute window — Python restatement (TEST INFRASTRUCTURE ONLY).

Only tests/ may import this module; the product planner lives in libspl
(paper_2205_05198_b200/csrc/window.cu) and is checked against it. Follows
/root/reference/proj/core/src/pipeline_sim.cpp:

  in_flight                  pipeline_sim.cpp:26-29
  rank_program               pipeline_sim.cpp:40-56
  microbatch_bytes           pipeline_sim.cpp:192-220 (extras: activation_memory.cpp:125-137)
  run_simulation (one rank)  pipeline_sim.cpp:222-275 (the per-rank byte walk; the cross-rank
                             tick assignment does not change a rank's own event order)
  microbatch_window_plan     pipeline_sim.cpp:297-359
  validate                   config.cpp:86-133

Exact arithmetic with fractions.Fraction (the reference uses Boost cpp_rational). Pinned to the
reference's own known answers (tests/test_pipeline_sim.cpp:257-362 and
acceptance_test.cpp:205-240): the p = 4, n_mb = 9 moving-window scenario stores microbatches
{1, 5, 9} on rank 0 with per-stage recompute counts 6, 6, 4, 0.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from . import KIND, per_layer_bytes_exact


class InfeasibleBudget(ValueError):
    def __init__(self, msg, min_feasible_budget):
        super().__init__(msg)
        self.min_feasible_budget = min_feasible_budget


@dataclass
class Model:
    heads: int
    hidden: int
    layers: int
    seq: int
    vocab: int
    tensor: int = 1
    pipeline: int = 1
    interleave: int = 1
    microbatch: int = 1
    microbatches: int = 1
    recompute: str = "selective"
    sequence_parallel: bool = True
    act_bytes: int = 2
    mask_bytes: int = 1
    logits_bytes: int = 4


def validate(m: Model):
    bad = []
    for f, v in (("a", m.heads), ("h", m.hidden), ("L", m.layers), ("s", m.seq), ("v", m.vocab),
                 ("t", m.tensor), ("p", m.pipeline), ("m", m.interleave), ("b", m.microbatch),
                 ("n_mb", m.microbatches)):
        if v < 1:
            bad.append(f)
    if not bad:
        if m.hidden % m.heads or m.hidden % m.tensor or m.seq % m.tensor:
            bad.append("div")
        if m.layers % (m.pipeline * m.interleave):
            bad.append("L")
        if m.microbatches < m.pipeline:
            bad.append("n_mb")
    if bad:
        raise ValueError(f"invalid configuration: {bad}")


def in_flight(p: int, stage: int) -> int:
    if stage < 0:
        raise ValueError("stage must be >= 0")
    return max(0, p - stage)


def rank_program(p: int, stage: int, n_mb: int):
    prog, fwd, bwd = [], 0, 0
    while fwd < p - stage:
        fwd += 1
        prog.append(("forward", fwd))
    while bwd < n_mb:
        bwd += 1
        prog.append(("backward", bwd))
        if fwd < n_mb:
            fwd += 1
            prog.append(("forward", fwd))
    return prog


def _per_layer(m: Model, kind: str) -> Fraction:
    n, d = per_layer_bytes_exact(m.heads, m.hidden, m.seq, m.microbatch, m.tensor, kind,
                                 m.sequence_parallel, m.act_bytes, m.mask_bytes)
    return Fraction(n, d)


def microbatch_bytes(m: Model, stage: int):
    """(fully_stored, checkpointed) bytes of one microbatch on pipeline rank `stage`."""
    validate(m)
    sbh = m.seq * m.microbatch * m.hidden
    extras = Fraction(0)
    if stage == 0:
        extras += Fraction(m.mask_bytes * sbh, m.tensor)
        if m.pipeline == 1:
            extras += Fraction(2 * m.act_bytes * sbh + m.logits_bytes * m.seq * m.microbatch * m.vocab,
                               m.tensor)
    lps = m.layers // m.pipeline
    full = int(_per_layer(m, "none") * lps + extras)  # floor (non-negative)
    ckpt = full if m.recompute == "none" else int(_per_layer(m, m.recompute) * lps + extras)
    return full, ckpt


def window_plan(m: Model, budget: int):
    validate(m)
    if m.recompute == "none":
        raise ValueError("window plan needs a full or selective inner strategy")
    p, n_mb = m.pipeline, m.microbatches
    sb = [microbatch_bytes(m, s) for s in range(p)]
    min_budget = max(in_flight(p, s) * sb[s][1] for s in range(p))
    if budget < min_budget:
        raise InfeasibleBudget(f"budget {budget} < {min_budget}", min_budget)
    modes = [[0] * n_mb for _ in range(p)]
    counts, recomputed = [], 0
    for s in range(p):
        full, ckpt = sb[s]
        slots, live, nf, nc = in_flight(p, s), 0, 0, 0
        for kind, mb in rank_program(p, s, n_mb):
            if kind == "forward":
                projected = (live + 1) * full + max(0, slots - (live + 1)) * ckpt
                if projected <= budget:
                    modes[s][mb - 1] = 1
                    live += 1
                    nf += 1
                else:
                    nc += 1
            elif modes[s][mb - 1]:
                live -= 1
        counts.append((nf, nc))
        recomputed += nc
    return {"modes": modes, "stage_counts": counts,
            "recomputed_fraction": Fraction(recomputed, p * n_mb),
            "min_feasible_budget": min_budget}


def stage_timeline(m: Model, stage: int, modes_row, dealloc: bool = True):
    """Bytes after each event of rank `stage` (recompute events included) and the peak."""
    full, ckpt = microbatch_bytes(m, stage)
    recompute = m.recompute != "none"
    out_tensor = m.act_bytes * m.seq * m.microbatch * m.hidden
    cur, peak, after = 0, 0, []
    for kind, mb in rank_program(m.pipeline, stage, m.microbatches):
        stored = full if modes_row[mb - 1] else ckpt
        if kind == "forward":
            cur += stored + (0 if dealloc else out_tensor)
        else:
            if recompute and not modes_row[mb - 1]:
                after.append(cur)
            cur -= stored + (0 if dealloc else out_tensor)
        after.append(cur)
        peak = max(peak, cur)
    return after, peak


assert KIND  # the kind names ("none", "full", "selective") are the ones oracle.KIND maps
