"""Microbatch-level recompute window on B200 (dev / measurement tool, GPU
box only): one pipeline rank of the 22B model (t = 1, L/p layers) runs its 1F1B program over
n_mb microbatches under window plans for a range of activation budgets, inner regime full or
selective. Per budget: the plan (microbatch_window_plan), the measured time of the whole rank
program (CUDA events on the caller stream, W warm-up runs), tokens/s, and the device's live
activation peak against the plan's simulated peak.

    python tools/window_bench.py [--layers 2] [--p 4] [--stage 0] [--n-mb 8] > out.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2, help="layers on this pipeline rank (L/p)")
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--stage", type=int, default=0)
    ap.add_argument("--n-mb", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--inner", default="full,selective")
    args = ap.parse_args()
    import torch
    import paper_2205_05198_b200 as spl
    torch.cuda.set_device(0)
    a, h, s, b = 64, 6144, 2048, 4  # 22B layer (BASELINE.json configs[1])
    for inner in args.inner.split(","):
        m = spl.ModelShape(heads=a, hidden=h, layers=args.layers * args.p, seq=s, vocab=51200,
                           tensor=1, pipeline=args.p, microbatch=b, microbatches=args.n_mb,
                           recompute=inner)
        full, ckpt = spl.microbatch_bytes(m, args.stage)
        lo = spl.window_plan(m, 2**63 - 1)["min_feasible_budget"]
        slots = args.p - args.stage
        budgets = [("all checkpointed (min)", lo)]
        for k in range(1, slots):
            budgets.append((f"{k} stored + {slots - k} checkpointed", k * full + (slots - k) * ckpt))
        budgets.append(("unbounded", 2**63 - 1))
        for label, budget in budgets:
            plan = spl.window_plan(m, budget)
            row = plan["modes"][args.stage]
            _, sim_peak = spl.stage_timeline(m, args.stage, row, True)
            cfg = spl.BlockConfig(a, h, s, b, dropout_p=0.1, causal=False, seed=42)
            w = spl.SeqparWindow(cfg, 1, args.layers, args.p, args.stage, row, recompute=inner)
            try:
                w.init_params(1234)
                g = torch.Generator(device="cuda:0").manual_seed(100)
                shp = w.shard_shape()
                mk = lambda: [[(torch.rand(shp, generator=g, device="cuda") * 2 - 1)  # noqa
                               .to(torch.bfloat16)] for _ in range(args.n_mb)]
                x, dy = mk(), mk()
                y = [[torch.empty_like(v[0])] for v in x]
                dx = [[torch.empty_like(v[0])] for v in x]
                for _ in range(args.warmup):
                    w.run(x, dy, y, dx)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.steps):
                    w.run(x, dy, y, dx)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.steps
                mem = w.memory()
                print(json.dumps({
                    "inner": inner, "budget_label": label, "budget_bytes": budget,
                    "p": args.p, "stage": args.stage, "n_mb": args.n_mb, "layers": args.layers,
                    "modes": row, "recomputed_fraction": str(plan["recomputed_fraction"]),
                    "ms_per_rank_program": ms, "ms_per_microbatch": ms / args.n_mb,
                    "tokens_per_s": args.n_mb * s * b / (ms / 1e3),
                    "microbatch_bytes": {"fully_stored": full, "checkpointed": ckpt},
                    "sim_peak_bytes": sim_peak, "device_live_peak_ledger": mem["live_peak_ledger"],
                    "slots": [mem["fully_stored_slots"], mem["checkpointed_slots"]],
                    "slots_ledger_bytes": mem["slots_ledger"],
                }), flush=True)
            finally:
                w.close()
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
