"""Table 4 of the paper on B200: forward / backward time of one 22B transformer layer for the
five experiments (no recompute TP / SP, full recompute, selective, selective + SP), with the
reference's FLOP model (paper_2205_05198_b200/report.py) turning the times into MFU / HFU.
Dev / measurement tool, GPU box only.

t = 1 runs the whole layer on one GPU. t > 1 runs the t ranks as simulated ranks on one GPU at
their true shard shapes; the per-GPU time is (measured - local-collective time) / t, i.e. the
compute of one rank of the real t-GPU group without its NVLink time (reported separately as the
NVLink-roofline time of the rank's collectives).

    python tools/layer_times.py --t 8 > gpurun_out/layer_times_t8.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# Per-GPU compute = step minus the collective class, so the simulated ranks use the
# collective-based reduce-scatter and all-gather (the NCCL ranks' default) unless told
# otherwise: fused, the slot reduction / shard reads run inside the consumers.
os.environ.setdefault("SPL_FUSED_RS", "0")
os.environ.setdefault("SPL_FUSED_AG", "0")

CONFIGS = {"22B": (64, 6144, 2048, 4), "175B": (96, 12288, 2048, 1), "530B": (128, 20480, 2048, 1),
           "1T": (160, 25600, 2048, 1)}


def measure(spl, torch, cfg, t, rc, sp, steps, warmup):
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
        for _ in range(warmup):
            L.forward(x, y)
            L.backward(dy, dx)
        torch.cuda.synchronize()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        for e in ev:
            e[0].record()
            L.forward(x, y)
            e[1].record()
            L.backward(dy, dx)
            e[2].record()
        torch.cuda.synchronize()
        fwd = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
        bwd = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
        comm = []
        for phase in ("fwd", "bwd"):
            L.profile(True)
            if phase == "fwd":
                L.forward(x, y)
            else:
                L.backward(dy, dx)
            comm.append(L.profile_read()["collective"]["ms"])
            L.profile(False)
            if phase == "fwd":
                L.backward(dy, dx)
            else:
                L.forward(x, y)
        return fwd, bwd, comm[0], comm[1]
    finally:
        L.close()
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="22B")
    ap.add_argument("--t", type=int, default=8)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_2205_05198_b200 as spl
    from paper_2205_05198_b200 import report as R
    torch.cuda.set_device(0)
    a, h, s, b = CONFIGS[args.config]
    t = args.t
    cfg = spl.BlockConfig(a, h, s, b, dropout_p=0.1, causal=False, seed=42)
    measured, raw = {}, {}
    for _, rc, sp, _, _ in R.TABLE4_ROWS:
        f, bw, cf, cb = measure(spl, torch, cfg, t, rc, sp, args.steps, args.warmup)
        measured[(rc, sp)] = ((f - cf) / t, (bw - cb) / t)
        raw[f"{rc}/sp={int(sp)}"] = {"fwd_ms_all_ranks": f, "bwd_ms_all_ranks": bw,
                                     "local_collective_ms": [cf, cb]}
    rows = R.table4(measured)
    shape = R.ModelShape(a, h, 1, s, 1)  # one layer; v = 1 (negligible; v = 0 is not a valid shape)
    peaks = {"nominal_bf16_2250": R.B200_NOMINAL_BF16}
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peaks["measured_bf16_sustained"] = int(pk["bf16_tflops_sustained"] * 1e12)
    except Exception:
        pass
    for r in rows:
        it = R.Fraction(r["combined_ms"]) / 1000
        r["flops_report"] = {k: R.flops_report(shape, b, r["recompute"], it, t, v)
                             for k, v in peaks.items()}
    print(json.dumps({"config": args.config, "t": t, "per_gpu": "compute of one rank (local "
                      "collectives excluded)" if t > 1 else "whole layer on one GPU",
                      "rows": rows, "raw": raw}, indent=1))


if __name__ == "__main__":
    main()
