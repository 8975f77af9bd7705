"""Layer fwd+bwd benchmark of the B200 sequence-parallel layer (arXiv 2205.05198 hot path).

    python bench.py --gpus N --steps K --warmup W            # our arm (t = N, one rank/GPU)
    python bench.py --impl reference --gpus N ...             # the reference CPU path

Workload (BASELINE.json configs[1]): the 22B-shape layer h=6144 a=64 s=2048 b=4, bf16,
dropout p=0.1, sequence parallel + selective recomputation, tensor-parallel degree t = N
(N=1: the whole layer on one GPU). A step = one layer forward + backward over one micro-batch
(s·b = 8192 tokens). value = tokens/s of the whole t-group = s·b / step time (max over ranks).
Inputs are synthetic (seeded U(-1,1)); params are LayerParams::random generated on the device.
The per-step working set (0.9 GB of weights alone at t=1) exceeds the 126 MB L2, so no
explicit flush is done between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # name: (heads, hidden, seq, batch)
    "tiny": (8, 256, 128, 2),
    "22B": (64, 6144, 2048, 4),
    "175B": (96, 12288, 2048, 1),
    "530B": (128, 20480, 2048, 1),
    "1T": (160, 25600, 2048, 1),
}
METRIC = "layer fwd+bwd tokens/s & MFU at t=1/2/4/8; activation bytes/GPU vs 34sbh/t"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def model_flops(a, h, s, b):
    # flops.cpp:29-34 x3 (fwd + bwd): 72 b s h^2 + 12 b s^2 h per layer (whole t-group)
    return 72.0 * b * s * h * h + 12.0 * b * s * s * h


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def share_unique_id(make_id, rank):
    """Rank 0 creates the NCCL unique id (libspl's spl_nccl_unique_id) and every rank gets
    it through torch.distributed (plumbing only; the data path is libspl's own NCCL comm)."""
    import torch.distributed as dist
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(value, device="cuda"):
    """Max of a per-rank float over the process group (timing = slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([float(value)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gemm_traffic_from_profile(cfg_name):
    """DRAM bytes per GEMM launch (read + write), averaged over the tcgen05 GEMM launches of
    one step, from the newest committed ncu capture (profiles/r0N_ncu_dram_<cfg>_t1_selective.json;
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum). None when absent."""
    prof = None
    for rnd in ("r02", "r01"):
        path = os.path.join(ROOT, "profiles", f"{rnd}_ncu_dram_{cfg_name}_t1_selective.json")
        try:
            prof = json.load(open(path))
            break
        except Exception:
            continue
    if prof is None:
        return None
    n = b = 0.0
    for k, v in prof.items():
        if k.startswith("gemm_tc"):
            n += v["launches"]
            b += v["launches"] * (v["dram_read_bytes_per_launch"] + v["dram_write_bytes_per_launch"])
    return b / n if n else None


def _layer_inputs(mod, cfg_name, s_sample, b_sample):
    a, h, _, _ = CONFIGS[cfg_name]
    import oracle as orc
    cfg = orc.BlockConfig(heads=a, hidden=h, seq=s_sample, batch=b_sample, dropout_p=0.1, seed=42)
    p = orc.params_random(h, 7)
    x = orc.random_uniform(1, (s_sample, b_sample, h), -1, 1)
    dy = orc.random_uniform(2, (s_sample, b_sample, h), -1, 1)
    return cfg, p, x, dy


def reference_cpu(cfg_name, s_sample, b_sample, budget_s, warmup=1, steps=1):
    """The reference's OWN seqpar fwd+bwd (block.cpp/tensor.cpp/collectives.cpp compiled
    unmodified into oracle/_ref/libref_seqpar.so — single-threaded, as the reference is) on a
    bounded sample of the workload: the config's full width (h, a) with s_sample·b_sample tokens.
    Falls back to the fp64 restatement (oracle port) on one thread when the library was not
    built. Returns (tokens/s, seconds per step, steps, warmup, kind)."""
    from oracle import ref as R
    import oracle as orc
    kind = "reference" if R.available() else "port"
    cfg, p, x, dy = _layer_inputs(None, cfg_name, s_sample, b_sample)
    if kind == "port":
        orc.set_threads(1)
        run = lambda: orc.seqpar_layer(cfg, 1, p, x, dy)  # noqa: E731
    else:
        run = lambda: R.seqpar_layer(cfg, 1, p, x, dy)  # noqa: E731
    t0 = time.perf_counter()
    run()  # first warm-up step, also sizes the run
    one = time.perf_counter() - t0
    fit = max(1, int(budget_s / max(one, 1e-3)) - 1)
    warmup = max(0, min(warmup - 1, fit // 2))
    steps = max(1, min(steps, fit - warmup))
    for _ in range(warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(steps):
        run()
    dt = (time.perf_counter() - t0) / steps
    return s_sample * b_sample / dt, dt, steps, warmup + 1, kind


def cpu_baseline_sample(cfg_name):
    """cpu_baseline of the ours-arm line (rank 0, N=1): the reference's own code on 1 core
    (faithful: the reference is single-threaded) on a 128-token sample, plus the fp64 port on
    all host cores on a 512-token sample (BASELINE.md §4 asks for both)."""
    import oracle as orc
    a, h, s, b = CONFIGS[cfg_name]
    s1 = s if cfg_name == "tiny" else 128
    b1 = b if cfg_name == "tiny" else 1
    v1, dt1, _, _, kind = reference_cpu(cfg_name, s1, b1, budget_s=60.0)
    s_all = s if cfg_name == "tiny" else 512
    b_all = b if cfg_name == "tiny" else 1
    cores = orc.set_threads(0)
    cfg, p, x, dy = _layer_inputs(None, cfg_name, s_all, b_all)
    t0 = time.perf_counter()
    orc.seqpar_layer(cfg, 1, p, x, dy)
    dta = time.perf_counter() - t0
    return {"value": v1, "unit": "tokens/s", "cores": 1, "kind": kind,
            "sample": f"the reference's own seqpar_block_forward+backward (fp64, oracle/_ref, "
                      f"1 thread) at h={h} a={a} s={s1} b={b1} t=1 ({dt1:.1f} s/step)",
            "all_cores": {"value": s_all * b_all / dta, "unit": "tokens/s", "cores": cores,
                          "kind": "port",
                          "sample": f"fp64 restatement (OpenMP) at h={h} a={a} s={s_all} "
                                    f"b={b_all} t=1 ({dta:.1f} s)"}}


def run_reference(args):
    """--impl reference: the reference's CPU path — its own block.cpp / tensor.cpp /
    collectives.cpp compiled unmodified (oracle/_ref, single-threaded like the reference) —
    rank 0 only, on a bounded sample of the config (full width, 256 tokens per step)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    a, h, s, b = CONFIGS[args.config]
    s_sample = s if args.config == "tiny" else 256
    b_sample = b if args.config == "tiny" else 1
    v, dt, steps, warmup, kind = reference_cpu(args.config, s_sample, b_sample, budget_s=240.0,
                                               warmup=args.warmup, steps=args.steps)
    who = ("the reference's own seqpar_block_forward+backward (block.cpp/tensor.cpp/"
           "collectives.cpp/rng.cpp compiled unmodified, oracle/_ref, Eigen/Boost shims)"
           if kind == "reference" else "fp64 restatement of the reference (oracle port)")
    sample = f"{who}, fp64, 1 thread, h={h} a={a} s={s_sample} b={b_sample} t=1, {steps} timed steps"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} layer fwd+bwd (sampled: {s_sample * b_sample} "
                                   f"tokens per step)", "heads": a, "hidden": h, "seq": s, "batch": b},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": 1, "kind": kind,
                             "sample": sample},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch(args):
    """`python bench.py --gpus N` (N > 1) without torchrun: re-exec under
    torch.distributed.run with one process per GPU — never a silent single-GPU run."""
    import socket
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        raise SystemExit(f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {n}")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="22B", choices=list(CONFIGS))
    ap.add_argument("--recompute", default="selective", choices=["none", "selective", "full"])
    ap.add_argument("--no-sp", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graphs", action="store_true")
    ap.add_argument("--dtype", default=None, choices=["bf16", "f32"],
                    help="compute dtype (default: f32 for the tiny config — BASELINE configs[0] "
                         "is quoted in fp32 — bf16 otherwise)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "ipc"],
                    help="transport of the t>1 collectives: NCCL, or libspl's CUDA-IPC peer-memory "
                         "transport (spl_create_ipc)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    import torch
    import paper_2205_05198_b200 as spl

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: one process per GPU")
    t = world
    torch.cuda.set_device(local_rank)
    dist = None
    nccl = None
    ipc = None
    if "WORLD_SIZE" in os.environ and "MASTER_ADDR" in os.environ:
        # launched by torchrun (any N, including 1): one rank per GPU; NCCL for the plumbing
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        if args.comm == "ipc" and t > 1:
            def exchange(hb):
                got = [None] * t
                dist.all_gather_object(got, hb)
                return got
            ipc = (rank, exchange)
        else:
            nccl = (rank, share_unique_id(spl.SeqparLayer.nccl_unique_id, rank))
    a, h, s, b = CONFIGS[args.config]
    sp = not args.no_sp
    cfg = spl.BlockConfig(a, h, s, b, dropout_p=0.1, causal=False, seed=42)
    dtype = args.dtype or ("f32" if args.config == "tiny" else "bf16")
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    L = spl.SeqparLayer(cfg, t, args.recompute, sp, dtype, device=local_rank,
                        check_finite=False, nccl=nccl, ipc=ipc)
    L.init_params(1234)
    L.set_graphs(not args.no_graphs)  # forward / backward replayed as CUDA graphs
    shp = L.shard_shape()
    gen = torch.Generator(device=f"cuda:{local_rank}").manual_seed(100 + rank)
    x = [(torch.rand(shp, generator=gen, device="cuda") * 2 - 1).to(tdt)]
    dy = [(torch.rand(shp, generator=gen, device="cuda") * 2 - 1).to(tdt)]
    y = [torch.empty_like(x[0])]
    dx = [torch.empty_like(x[0])]

    def step():
        L.forward(x, y)
        L.backward(dy, dx)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 1)):
        step()
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    L.launch_count(reset=True)
    # device-timed region on the layer's stream (forward/backward join the caller stream)
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(args.steps):
        step()
    stop.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    launches = L.launch_count(reset=True)
    clk = clocks.stop()
    ms = max_over_ranks(ms)
    ms_step = ms / args.steps
    tokens = s * b
    value = tokens / (ms_step / 1e3)

    # per-kernel-class times: a second pass with events around every launch
    barrier()
    L.profile(True)
    for _ in range(args.steps):
        step()
    prof = L.profile_read()
    L.profile(False)

    # end-to-end through the host-buffer C-ABI step (H2D x, dy and D2H y, dx every step), the
    # way a training loop drives it: spl_step_host_async over two pinned host buffer sets, the
    # copies of one step overlapping the compute of its neighbours, one wait at the end.
    e2e = None
    if not args.no_e2e:
        nbytes = x[0].numel() * x[0].element_size()
        hx = [x[0].cpu().pin_memory() for _ in range(2)]
        hdy = [dy[0].cpu().pin_memory() for _ in range(2)]
        hy = [torch.empty_like(hx[0]).pin_memory() for _ in range(2)]
        hdx = [torch.empty_like(hx[0]).pin_memory() for _ in range(2)]
        for j in range(2):
            L.step_host(hx[j], hdy[j], hy[j], hdx[j])
        barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            j = i & 1
            L.step_host_async(hx[j], hdy[j], hy[j], hdx[j])
        L.step_host_wait()
        el = time.perf_counter() - t0
        el = max_over_ranks(el)
        e2e = {"value": tokens / (el / args.steps), "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * nbytes, "d2h_bytes_per_step": 2 * nbytes,
               "path": "spl_step_host_async (pinned, double-buffered host sets), host wall clock"}

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    pk, pk_kind = peaks()
    g = prof["gemm"]
    gemm_tflops = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else 0.0
    burst = pk.get("bf16_tflops")
    sustained = pk.get("bf16_tflops_sustained", burst)
    hbm = pk.get("hbm_gbs")
    total_prof_ms = sum(v["ms"] for v in prof.values())
    led, phys, unc = L.saved_bytes(0)
    mf = model_flops(a, h, s, b)

    def cls_roof(name, bound):
        v = prof[name]
        if not v["ms"]:
            return None
        if bound == "tensor":
            ach = v["flops"] / (v["ms"] / 1e3) / 1e12
            return {"bound": "tensor", "achieved": ach, "peak": burst, "unit": "TFLOP/s",
                    "frac": ach / burst if burst else None, "ms_per_step": v["ms"] / args.steps}
        ach = v["bytes"] / (v["ms"] / 1e3) / 1e9
        peak_b = hbm if bound == "hbm" else 900.0  # NVLink 5: 900 GB/s per direction
        return {"bound": bound, "achieved": ach, "peak": peak_b, "unit": "GB/s",
                "frac": ach / peak_b if peak_b else None, "ms_per_step": v["ms"] / args.steps}

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic (seeded U(-1,1) inputs, LayerParams::random on device)",
        "config": {"workload": f"{args.config}-shape layer fwd+bwd, t={t}, SP={'on' if sp else 'off'}, "
                               f"{args.recompute} recompute",
                   "heads": a, "hidden": h, "seq": s, "batch": b, "t": t, "dropout_p": 0.1,
                   "causal": False, "parallelism": f"tp{t}+sp" if sp else f"tp{t}",
                   "comm": (args.comm if t > 1 else "none"),
                   "collectives": L.comm_paths() if t > 1 else None,
                   "l2": "working set > L2 (weights alone 0.9 GB/t); no flush"},
        "mfu": mf / (ms_step / 1e3) / t / (burst * 1e12),
        "mfu_vs_sustained_peak": mf / (ms_step / 1e3) / t / (sustained * 1e12),
        "mfu_vs_nominal_2250": mf / (ms_step / 1e3) / t / 2.25e15,
        "activation_bytes_per_gpu": {"ledger": led, "physical": phys, "uncounted_stats": unc,
                                     "formula_34sbh_over_t": 34 * s * b * h // t,
                                     "per_layer_bytes": spl.per_layer_bytes(a, h, s, b, t, args.recompute, sp)},
        "roofline": {"kernel": "tcgen05 GEMM (all layer GEMMs)", "bound": "tensor",
                     "achieved": gemm_tflops, "peak": burst, "unit": "TFLOP/s",
                     "frac": gemm_tflops / burst if burst else None,
                     "traffic": gemm_traffic_from_profile(args.config) if t == 1 else None,
                     "traffic_unit": "DRAM bytes per GEMM launch (ncu, profiles/)",
                     "algorithmic_bytes_per_launch": g["bytes"] / max(g["launches"], 1),
                     "peak_kind": f"{pk_kind} bf16_tflops (burst: cuBLAS 8192^3 best of 10)",
                     "frac_of_sustained_peak": gemm_tflops / sustained if sustained else None,
                     "share_of_step": g["ms"] / total_prof_ms if total_prof_ms else None},
        "rooflines": {"gemm": cls_roof("gemm", "tensor"), "attention": cls_roof("attention", "tensor"),
                      "elementwise": cls_roof("elementwise", "hbm"),
                      "collective": cls_roof("collective", "nvlink") if t > 1 else None,
                      "other": ({"what": "softmax-dropout keep-bit RNG (ALU-bound: 2 splitmix64 "
                                         "per interior element)",
                                 "ms_per_step": prof["other"]["ms"] / args.steps,
                                 "keys_per_s": (a // t) * b * s * s * prof["other"]["launches"] / args.steps
                                 / max(prof["other"]["ms"] / args.steps / 1e3, 1e-12)}
                                if prof["other"]["ms"] else None)},
        "kernel_classes": {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                               "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] and v["flops"] else None,
                               "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] and v["bytes"] else None}
                           for k, v in prof.items()},
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": e2e,
    }
    if args.gpus == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline_sample(args.config)
        cb.pop("seconds", None)
        line["cpu_baseline"] = cb
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
