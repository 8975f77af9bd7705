"""Render tools/sweep.py output (JSON lines) as the markdown table in profiles/ (dev tool)."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
base = {}
for d in rows:
    if d.get("recompute") == "none" and "error" not in d:
        base[(d["config"], d["t"], d["sp"])] = d["per_gpu_compute_ms"]
print("| config | t | regime | SP | per-GPU compute ms | tokens/s (t-group, compute) | MFU (nominal 2.25 PF) "
      "| GEMM TFLOP/s | attn ms | RNG ms | elementwise ms | vs none | ledger B/GPU | per_layer_bytes | = |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for d in rows:
    if "error" in d:
        print(f"| {d['config']} | {d['t']} | {d['recompute']} | {d['sp']} | error: {d['error'][:60]} |")
        continue
    c = d["class_ms_per_gpu"]
    nb = base.get((d["config"], d["t"], d["sp"]))
    rel = f"{d['per_gpu_compute_ms'] / nb - 1:+.1%}" if nb else "—"
    eq = "yes" if d["ledger_bytes"] == d["per_layer_bytes"] else "phys<ref (full: A·sbh/t held)"
    print(f"| {d['config']} | {d['t']} | {d['recompute']} | {'on' if d['sp'] else 'off'} | "
          f"{d['per_gpu_compute_ms']:.2f} | {d['tokens_per_s_group_compute_only']:,.0f} | "
          f"{d['mfu_vs_nominal_2250']:.3f} | {d['gemm_tflops']:.0f} | {c['attention']:.2f} | "
          f"{c['other']:.2f} | {c['elementwise']:.2f} | {rel} | {d['ledger_bytes']:,} | "
          f"{d['per_layer_bytes']:,} | {eq} |")
