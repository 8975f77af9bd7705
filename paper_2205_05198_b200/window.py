"""Microbatch-level recompute window over the C ABI.

Mirrors the reference's pipeline API (/root/reference/proj/core/include/actplan/
pipeline_sim.hpp): microbatch_window_plan (108-110), in_flight (46), the per-rank part of
simulate_memory_with_modes (79-83) and InfeasibleBudgetError (98-103, here InfeasibleBudget
with .min_feasible_budget). Errors: std::invalid_argument -> ValueError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction

from . import _lib
from ._lib import check, lib


class InfeasibleBudget(ValueError):
    def __init__(self, msg: str, min_feasible_budget: int):
        super().__init__(msg)
        self.min_feasible_budget = min_feasible_budget


@dataclass
class ModelShape:
    """ModelShape + ParallelLayout (without d) + inner RecomputeStrategy + ByteConvention."""
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

    def c(self) -> _lib.ModelDesc:
        d = _lib.ModelDesc()
        lib().spl_model_desc_default(C.byref(d))
        for f in ("heads", "hidden", "layers", "seq", "vocab", "tensor", "pipeline", "interleave",
                  "microbatch", "microbatches", "act_bytes", "mask_bytes", "logits_bytes"):
            setattr(d, f, int(getattr(self, f)))
        if self.recompute not in _lib.RECOMPUTE:
            raise ValueError(f"unknown recompute kind {self.recompute!r}")
        d.recompute = _lib.RECOMPUTE[self.recompute]
        d.sequence_parallel = int(bool(self.sequence_parallel))
        return d


def in_flight(p: int, stage: int) -> int:
    if stage < 0:
        raise ValueError("stage must be >= 0")
    return max(0, p - stage)


def microbatch_bytes(m: ModelShape, stage: int) -> tuple[int, int]:
    full, ckpt = C.c_int64(), C.c_int64()
    check(lib().spl_microbatch_bytes(C.byref(m.c()), stage, C.byref(full), C.byref(ckpt)))
    return full.value, ckpt.value


def window_plan(m: ModelShape, budget: int) -> dict:
    p, n = m.pipeline, m.microbatches
    modes = (C.c_uint8 * max(1, p * n))()
    counts = (C.c_int64 * max(2, 2 * p))()
    num, den, minb = C.c_int64(), C.c_int64(), C.c_int64()
    budget = min(int(budget), 2**63 - 1)
    rc = lib().spl_window_plan(C.byref(m.c()), budget, modes, counts, C.byref(num), C.byref(den),
                               C.byref(minb))
    if rc == _lib.SPL_EBUDGET:
        raise InfeasibleBudget(lib().spl_last_error().decode(), minb.value)
    check(rc)
    return {"modes": [[modes[s * n + i] for i in range(n)] for s in range(p)],
            "stage_counts": [(counts[2 * s], counts[2 * s + 1]) for s in range(p)],
            "recomputed_fraction": Fraction(num.value, den.value),
            "min_feasible_budget": minb.value}


def stage_timeline(m: ModelShape, stage: int, modes_row, dealloc: bool = True):
    """Bytes held by rank `stage` after each event of its program, and the peak."""
    n = m.microbatches
    row = (C.c_uint8 * max(1, n))(*[1 if v else 0 for v in modes_row])
    cap = 3 * n + 1
    out = (C.c_int64 * cap)()
    ne, peak = C.c_int64(), C.c_int64()
    check(lib().spl_stage_timeline(C.byref(m.c()), stage, row, int(dealloc), out, cap,
                                   C.byref(ne), C.byref(peak)))
    return [out[i] for i in range(ne.value)], peak.value


class SeqparWindow:
    """Window executor (spl_window_*): pipeline rank `stage` of p running its 1F1B program over
    len(modes_row) microbatches with `layers` layers on t simulated ranks; modes_row[i] = 1 keeps
    microbatch i+1 fully stored (no recompute), 0 checkpoints it under cfg's inner regime.
    Gradients accumulate over the microbatches; layers(l) gives the parameter / gradient view."""

    def __init__(self, cfg, t: int, layers: int, p: int, stage: int, modes_row,
                 recompute: str = "selective", sequence_parallel: bool = True,
                 dtype: str = "bf16", device: int = 0, check_finite: bool = False):
        from .seqpar import BlockConfig, SeqparLayer, _desc
        self.cfg, self.t, self.dtype, self.device = cfg, t, dtype, device
        self.n_mb = len(modes_row)
        d = _desc(cfg, recompute, sequence_parallel, dtype, check_finite)
        row = (C.c_uint8 * self.n_mb)(*[1 if v else 0 for v in modes_row])
        self._w = C.c_void_p()
        check(lib().spl_window_create_local(C.byref(d), device, t, layers, p, stage, self.n_mb,
                                            row, C.byref(self._w)))
        self.layers = []
        for l in range(layers):
            h = C.c_void_p()
            check(lib().spl_window_layer(self._w, l, C.byref(h)))
            cl = BlockConfig(**{**cfg.__dict__, "layer_index": cfg.layer_index + l})
            self.layers.append(SeqparLayer(cl, t, recompute, sequence_parallel, dtype, device,
                                           check_finite, _borrow=h))
        self.local = self.layers[0].local

    def close(self):
        for L in getattr(self, "layers", []):
            L.close()
        if getattr(self, "_w", None):
            lib().spl_window_destroy(self._w)
            self._w = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard_shape(self):
        return self.layers[0].shard_shape()

    def init_params(self, seed: int):
        for L in self.layers:
            L.init_params(seed)

    def run(self, x: list, dy: list, y: list | None = None, dx: list | None = None):
        """x, dy: n_mb lists of local-rank device shards. Returns (y, dx) in the same layout."""
        import torch
        check(lib().spl_window_set_stream(
            self._w, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))
        if len(x) != self.n_mb or len(dy) != self.n_mb:
            raise ValueError("expected one shard list per microbatch")
        if y is None:
            y = [[torch.empty_like(a) for a in mb] for mb in x]
        if dx is None:
            dx = [[torch.empty_like(a) for a in mb] for mb in x]

        def arr(ts):
            flat = [a for mb in ts for a in mb]
            if len(flat) != self.n_mb * self.local:
                raise ValueError("expected one shard per rank")
            return (C.c_void_p * len(flat))(*[a.data_ptr() for a in flat])
        check(lib().spl_window_run(self._w, arr(x), arr(dy), arr(y), arr(dx)))
        return y, dx

    def memory(self) -> dict:
        out = (C.c_int64 * 6)()
        check(lib().spl_window_memory(self._w, out))
        keys = ["fully_stored_slots", "checkpointed_slots", "slots_ledger", "live_peak_ledger",
                "params_and_grads", "workspace"]
        return dict(zip(keys, list(out)))
