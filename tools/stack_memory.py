"""Measured device memory of an L-layer stack vs the accountant (dev /
measurement tool, GPU box only).

For each regime: build an L-layer stack (one workspace, per-layer saved activations), run
W + K fwd+bwd steps, and report
  * the driver's view: cudaMemGetInfo used-bytes delta from before the stack was created, at the
    peak after the timed steps (the stack allocates everything up front, so this is the peak);
  * the library's view: Σ ledger (reference convention), physical saved, uncounted saved
    (LN stats / LSE), shared workspace, params, grads (spl_stack_memory);
  * total_first_stage_bytes(p = 1) and the paper's 34·sbh/t · L (SP + selective);
  * the step time and tokens/s of the L-layer fwd+bwd.

    python tools/stack_memory.py [--config 22B] [--layers 8] [--t 1] > gpurun_out/stack.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {"tiny": (8, 256, 128, 2), "22B": (64, 6144, 2048, 4), "175B": (96, 12288, 2048, 1),
           "530B": (128, 20480, 2048, 1), "1T": (160, 25600, 2048, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="22B")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--t", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--regimes", default="none,selective,full")
    args = ap.parse_args()
    import torch
    import paper_2205_05198_b200 as spl
    torch.cuda.set_device(0)
    a, h, s, b = CONFIGS[args.config]
    L, t = args.layers, args.t
    for rc in args.regimes.split(","):
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        free0, total = torch.cuda.mem_get_info()
        cfg = spl.BlockConfig(a, h, s, b, dropout_p=0.1, causal=False, seed=42)
        st = spl.SeqparStack(cfg, t, L, rc, True, "bf16", check_finite=False)
        for l in range(L):
            st.layers[l].init_params(1234 + l)
            st.layers[l].set_graphs(True)
        shp = st.shard_shape()
        g = torch.Generator(device="cuda:0").manual_seed(100)
        x = [(torch.rand(shp, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(t)]
        dy = [(torch.rand(shp, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(t)]
        y = [torch.empty_like(x[0]) for _ in range(t)]
        dx = [torch.empty_like(x[0]) for _ in range(t)]
        io_bytes = 4 * t * x[0].numel() * 2
        for _ in range(args.warmup):
            st.forward(x, y)
            st.backward(dy, dx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            st.forward(x, y)
            st.backward(dy, dx)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        free1, _ = torch.cuda.mem_get_info()
        m = st.memory(0)
        tfs = spl.total_first_stage_bytes(a, h, s, b, t, rc, True, L)
        out = {
            "config": args.config, "t": t, "layers": L, "recompute": rc, "sp": True,
            "ms_per_step": ms, "tokens_per_s": s * b / (ms / 1e3),
            "ms_per_layer": ms / L,
            "device_used_bytes": free0 - free1,
            "device_used_minus_io": free0 - free1 - io_bytes,
            "library": m,
            "library_total": sum(v for k, v in m.items() if k != "ledger"),
            "total_first_stage_bytes": tfs,
            "ledger_equals_total_first_stage": m["ledger"] == tfs,
            "paper_34sbh_over_t_times_L": 34 * s * b * h // t * L,
        }
        print(json.dumps(out), flush=True)
        st.close()
        del x, dy, y, dx


if __name__ == "__main__":
    main()
