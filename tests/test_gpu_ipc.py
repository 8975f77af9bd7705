"""libspl's one-rank-per-process schedule, executed: two processes share cuda:0 as a t=2
group over the CUDA-IPC transport (spl_ipc_open / spl_create_ipc). Every collective goes
through IPC-mapped peer memory sequenced by the device barrier, and the reduce-scatter fused
into the row-parallel GEMMs lands in the peer's slots with the arrival / generation counters
and the producer-side back-pressure wait — the code an 8-GPU NVLink group runs.

Done means bit-identity with spl_create_local(t=2) (the simulated-rank harness) on the same
inputs: y and dx shards, every parameter gradient and the CommLog counters.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from test_gpu_layer import spl  # noqa: F401

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

SMALL = dict(heads=8, hidden=256, seq=128, batch=2)       # head_dim 32
UMMA = dict(heads=4, hidden=256, seq=256, batch=2)        # head_dim 64, RL % 128 == 0
WIDE = dict(heads=4, hidden=512, seq=256, batch=2)        # h/t = 256: the pulled all-gather
CASES = [
    dict(shape=UMMA, recompute="selective", dtype="bf16"),                 # fused RS (default)
    dict(shape=UMMA, recompute="none", dtype="bf16", env={"SPL_FUSED_RS": "0"}),  # pushed RS
    # all-gathers fused into the consuming GEMMs, which pull the peer's shards from its memory
    # (default at this width), with the fused reduce-scatter; then the pushed all-gather
    dict(shape=WIDE, recompute="selective", dtype="bf16"),
    dict(shape=WIDE, recompute="none", dtype="bf16", graphs=True, steps=3),
    dict(shape=WIDE, recompute="selective", dtype="bf16", env={"SPL_FUSED_AG": "0"}),
    dict(shape=WIDE, recompute="full", dtype="bf16", causal=True),  # pulled AG, forward re-run
    dict(shape=SMALL, recompute="full", dtype="f32", causal=True),
    dict(shape=SMALL, recompute="selective", dtype="bf16", sp=False),      # f̄ all-reduce
    dict(shape=UMMA, recompute="selective", dtype="bf16", graphs=True, steps=3),  # graph replays
]


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_local(spl, orc, case):
    import torch
    sh = case["shape"]
    s, b, h = sh["seq"], sh["batch"], sh["hidden"]
    cfg = spl.BlockConfig(sh["heads"], h, s, b, 0.1, case.get("causal", False), 42)
    x = orc.random_uniform(orc.hash_counter(42, 1000), (s, b, h), -1, 1)
    dy = orc.random_uniform(orc.hash_counter(42, 2000), (s, b, h), -1, 1)
    p = orc.params_random(h, orc.hash_counter(42, 3000))
    sp = case.get("sp", True)
    L = spl.SeqparLayer(cfg, 2, case["recompute"], sp, case["dtype"], device=0)
    L.load_params(p)
    td = torch.float32 if case["dtype"] == "f32" else torch.bfloat16
    if sp:
        xd = [torch.from_numpy(np.ascontiguousarray(v)).to("cuda", td) for v in np.split(x, 2, 0)]
        dd = [torch.from_numpy(np.ascontiguousarray(v)).to("cuda", td) for v in np.split(dy, 2, 0)]
    else:
        xd = [torch.from_numpy(x).to("cuda", td) for _ in range(2)]
        dd = [torch.from_numpy(dy).to("cuda", td) for _ in range(2)]
    y = L.forward(xd)
    dx = L.backward(dd)
    torch.cuda.synchronize()
    out = dict(y=[v.double().cpu().numpy() for v in y], dx=[v.double().cpu().numpy() for v in dx],
               grads=L.grads(), w1=[L.w1_grad_shard(r) for r in range(2)], comm=L.comm_log(),
               paths=L.comm_paths())
    L.close()
    return out


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(
    [c["recompute"], c["dtype"]] + [k for k in ("causal", "graphs") if c.get(k)] +
    (["sp_off"] if c.get("sp") is False else []) + [f"{k}={v}" for k, v in c.get("env", {}).items()]))
def test_two_processes_bit_identical_to_local(spl, orc, tmp_path, case):
    env = dict(os.environ, **case.get("env", {}))
    port = str(free_port())
    outs = [str(tmp_path / f"r{r}.npz") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "ipc_worker.py"), str(r), port,
                               outs[r], json.dumps({k: v for k, v in case.items() if k != "env"})],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(2)]
    logs = []
    for pr in procs:
        try:
            logs.append(pr.communicate(timeout=240)[0])
        except subprocess.TimeoutExpired:
            pr.kill()
            logs.append(pr.communicate()[0])
    for pr, lg in zip(procs, logs):
        assert pr.returncode == 0, lg[-3000:]
    got = [np.load(o) for o in outs]
    os.environ.update(case.get("env", {}))
    try:
        want = run_local(spl, orc, case)
    finally:
        for k in case.get("env", {}):
            os.environ.pop(k, None)
    sp = case.get("sp", True)
    # the paths the peer ranks ran: the pulled all-gather wherever the simulated group fuses it
    # (same eligibility), unless switched off
    for r in range(2):
        fused_rs, ag = got[r]["paths"]
        assert bool(fused_rs) == want["paths"]["fused_rs"], (r, got[r]["paths"], want["paths"])
        assert ("copy", "local", "pull")[ag] == ("pull" if want["paths"]["all_gather"] == "local"
                                                 else "copy"), (r, got[r]["paths"], want["paths"])
    if case["shape"] is WIDE and "SPL_FUSED_AG" not in case.get("env", {}):
        assert want["paths"]["all_gather"] == "local" and got[0]["paths"][1] == 2
    for r in range(2):
        assert np.array_equal(got[r]["y"], want["y"][r]), f"y rank {r}"
        assert np.array_equal(got[r]["dx"], want["dx"][r]), f"dx rank {r}"
        assert np.array_equal(got[r]["w1"], want["w1"][r]), f"w1 shard rank {r}"
    # sharded gradients: each rank fills its own shard (disjoint); replicated ones all-reduced
    h = case["shape"]["hidden"]
    import oracle as orc_mod
    G = [orc_mod.unpack(h, g["grads"]) for g in got]
    W = orc_mod.unpack(h, want["grads"])
    for name in W:
        if name in ("bo", "b2", "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias"):
            for r in range(2):
                assert np.array_equal(G[r][name], W[name]), (name, r)
        else:
            assert np.array_equal(G[0][name] + G[1][name], W[name]), name
    # CommLog: same counts of the same collectives per rank as the simulated group
    wc = np.array([[v["all_gathers"], v["reduce_scatters"], v["all_reduces"], v["ring_elements"]]
                   for v in want["comm"].values()])
    steps = case.get("steps", 1)  # CUDA-graph replays add the captured increments per launch
    for r in range(2):
        assert np.array_equal(got[r]["comm"], steps * wc), (got[r]["comm"], wc)
