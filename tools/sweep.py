"""Per-layer sweep over BASELINE.json's configs (dev/measurement tool, GPU box only).

For every (config, t, recompute, SP) case: one layer handle, LayerParams::random on the device,
seeded U(-1,1) inputs, W warm-up steps, K timed fwd+bwd steps (CUDA events on the caller
stream), then a profiled pass for the per-kernel-class split, plus the activation ledger.

t > 1 runs the t ranks of the group as *simulated ranks on one GPU* (spl_create_local): each
rank's program runs at its true shard shapes (GEMM K = h/t, a/t heads, s/t-row shards) and the
collectives become device copies / rank-ordered sums. The per-GPU compute time of one rank is
then (step - collective-class time) / t; the NVLink time of the real t-GPU group is not in it
(see 'comm_model_ms', the §8(d) NVLink-roofline time of that rank's 10 AG/RS ops).

    python tools/sweep.py [--quick] > gpurun_out/sweep.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# Per-GPU compute = step minus the collective class, so the simulated ranks use the
# collective-based reduce-scatter and all-gather (the NCCL ranks' default) unless told
# otherwise: fused, the slot reduction / shard reads run inside the consumers.
os.environ.setdefault("SPL_FUSED_RS", "0")
os.environ.setdefault("SPL_FUSED_AG", "0")

CONFIGS = {"tiny": (8, 256, 128, 2), "22B": (64, 6144, 2048, 4), "175B": (96, 12288, 2048, 1),
           "530B": (128, 20480, 2048, 1), "1T": (160, 25600, 2048, 1)}
NVLINK_GBS = 900.0  # per direction, NVLink 5 (B200)


def cases(quick: bool):
    out = []
    for rc in ("none", "selective", "full"):
        out.append(("22B", 1, rc, True))
    for rc in ("none", "selective", "full"):
        out.append(("22B", 8, rc, True))
    out.append(("22B", 8, "selective", False))
    if quick:
        return out
    for t in (1, 2, 4, 8):
        for rc in ("none", "selective", "full"):
            for sp in ((True,) if t == 1 else (True, False)):
                out.append(("175B", t, rc, sp))
    for rc in ("none", "selective", "full"):
        out.append(("530B", 8, rc, True))
    for rc in ("selective", "full"):
        out.append(("1T", 8, rc, True))
    out.append(("1T", 1, "selective", True))
    return out


def run_case(spl, torch, name, t, rc, sp, steps, warmup):
    a, h, s, b = CONFIGS[name]
    cfg = spl.BlockConfig(a, h, s, b, dropout_p=0.1, causal=False, seed=42)
    L = spl.SeqparLayer(cfg, t, rc, sp, "bf16", device=0, check_finite=False)
    try:
        L.init_params(1234)
        L.set_graphs(True)
        shp = L.shard_shape()
        g = torch.Generator(device="cuda:0").manual_seed(100)
        x = [(torch.rand(shp, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(t)]
        dy = [(torch.rand(shp, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(t)]
        y = [torch.empty_like(x[0]) for _ in range(t)]
        dx = [torch.empty_like(x[0]) for _ in range(t)]

        def step():
            L.forward(x, y)
            L.backward(dy, dx)

        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        L.profile(True)
        for _ in range(steps):
            step()
        prof = L.profile_read()
        L.profile(False)
        led, phys, unc = L.saved_bytes(0)
        peak_mem = torch.cuda.max_memory_allocated()
        mf = 72.0 * b * s * h * h + 12.0 * b * s * s * h
        comm_ms = prof["collective"]["ms"] / steps
        per_gpu_ms = (ms - comm_ms) / t
        # NVLink roofline of one rank's 8 AG/RS + 2 re-gathers (N = 2sbh bytes each, (t-1)/t)
        nbytes = 2.0 * s * b * h
        n_ops = 10 if (sp and rc != "full") else (14 if sp else 8)
        comm_model_ms = n_ops * nbytes * (t - 1) / t / (NVLINK_GBS * 1e9) * 1e3 if t > 1 else 0.0
        gemm = prof["gemm"]
        return {
            "config": name, "t": t, "recompute": rc, "sp": sp, "heads": a, "hidden": h, "seq": s,
            "batch": b, "steps": steps, "ms_per_step_all_ranks": ms,
            "per_gpu_compute_ms": per_gpu_ms,
            "tokens_per_s_group_compute_only": s * b / (per_gpu_ms / 1e3),
            "comm_model_ms_nvlink": comm_model_ms,
            "mfu_vs_nominal_2250": mf / t / (per_gpu_ms / 1e3) / 2.25e15,
            "gemm_tflops": gemm["flops"] / (gemm["ms"] / 1e3) / 1e12 if gemm["ms"] else None,
            "class_ms_per_gpu": {k: v["ms"] / steps / t for k, v in prof.items()},
            "ledger_bytes": led, "physical_bytes": phys, "uncounted_stats_bytes": unc,
            "per_layer_bytes": spl.per_layer_bytes(a, h, s, b, t, rc, sp),
            "formula_34sbh_over_t": 34 * s * b * h // t if sp else None,
            "formula_sp_none": (34 * s * b * h // t + 5 * a * s * s * b // t) if sp else None,
            "peak_allocated_bytes_torch": peak_mem,
        }
    finally:
        L.close()
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default=None, help="comma list of config names")
    args = ap.parse_args()
    import torch
    import paper_2205_05198_b200 as spl
    torch.cuda.set_device(0)
    for name, t, rc, sp in cases(args.quick):
        if args.only and name not in args.only.split(","):
            continue
        t0 = time.time()
        try:
            r = run_case(spl, torch, name, t, rc, sp, args.steps, args.warmup)
        except Exception as e:  # keep sweeping; record the failure
            r = {"config": name, "t": t, "recompute": rc, "sp": sp, "error": repr(e)}
        r["wall_s"] = time.time() - t0
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
