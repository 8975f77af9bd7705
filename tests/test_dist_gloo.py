"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path.

1. bench.py's distributed plumbing: rank-0 NCCL-id broadcast, barrier, max-over-ranks timing.
2. The per-rank program of the NCCL handle (one process per rank; g/ḡ as all-gather /
   reduce-scatter of contiguous sequence chunks, the six replicated-gradient all-reduces),
   restated on the oracle primitives with real torch.distributed collectives, must equal the
   single-process simulated-rank oracle (block.cpp:512-749 with rank-ordered sums).
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, fn, *args):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    import sys

    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def _plumbing(rank, world):
    import torch
    import torch.distributed as dist

    import bench
    uid = bench.share_unique_id(lambda: bytes(range(128)) if rank == 0 else None, rank)
    assert uid == bytes(range(128))
    v = bench.max_over_ranks(float(rank + 1), device="cpu")
    assert v == float(world)
    dist.barrier()


def test_bench_plumbing_two_ranks():
    _run(2, _plumbing)


def _seqpar_rank_program(rank, world, out_dir):
    """Rank `rank` of a `world`-way TP+SP layer with gloo collectives (fwd + bwd)."""
    import torch
    import torch.distributed as dist

    import oracle as orc
    cfg = orc.BlockConfig(heads=4, hidden=16, seq=8, batch=2, dropout_p=0.1, seed=42)
    t, s, b, h = world, cfg.seq, cfg.batch, cfg.hidden
    x = orc.random_uniform(orc.hash_counter(42, 1000), (s, b, h), -1, 1)
    dy = orc.random_uniform(orc.hash_counter(42, 2000), (s, b, h), -1, 1)
    P = orc.params_random(h, orc.hash_counter(42, 3000))
    W = orc.unpack(h, P)
    RL, lw, fw, lh, hd = (s // t) * b, h // t, 4 * h // t, cfg.heads // t, h // cfg.heads
    p = cfg.dropout_p
    inv = 1.0 / (1.0 - p)

    def ag(shard):  # g: all-gather contiguous sequence chunks
        parts = [torch.zeros_like(torch.from_numpy(shard)) for _ in range(t)]
        dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(shard)))
        return torch.cat(parts).numpy()

    def rs(full):  # ḡ: reduce-scatter into contiguous sequence chunks
        out = torch.zeros((RL, full.shape[1]), dtype=torch.float64)
        dist.reduce_scatter(out, list(torch.from_numpy(np.ascontiguousarray(full)).chunk(t)))
        return out.numpy()

    def mask(op):
        key = orc.mask_key_fold(cfg.seed, 0, op, 1)
        full = orc.dropout_mask(key, s * b * h, p).reshape(s * b, h)
        return full[rank * RL:(rank + 1) * RL]

    def ln(v, g, be):
        mu = v.mean(1, keepdims=True)
        var = ((v - mu) ** 2).mean(1, keepdims=True)
        iv = 1 / np.sqrt(var + cfg.layer_norm_eps)
        return (v - mu) * iv * g + be, mu, iv

    def ln_bwd(dyv, v, mu, iv, g):
        xh = (v - mu) * iv
        dxh = dyv * g
        dx = iv * (dxh - dxh.mean(1, keepdims=True) - xh * (dxh * xh).mean(1, keepdims=True))
        return dx, (dyv * xh).sum(0), dyv.sum(0)

    from scipy.special import erf
    gelu = lambda z: 0.5 * z * (1 + erf(z / np.sqrt(2)))
    dgelu = lambda z: 0.5 * (1 + erf(z / np.sqrt(2))) + z * np.exp(-0.5 * z * z) / np.sqrt(2 * np.pi)
    cs = lambda k: slice(rank * k, (rank + 1) * k)

    xs = x.reshape(s * b, h)[rank * RL:(rank + 1) * RL]
    y1, mu1, iv1 = ln(xs, W["ln1_gain"], W["ln1_bias"])
    Y1 = ag(y1)
    q = Y1 @ W["wq"][:, cs(lw)] + W["bq"][cs(lw)]
    k = Y1 @ W["wk"][:, cs(lw)] + W["bk"][cs(lw)]
    v = Y1 @ W["wv"][:, cs(lw)] + W["bv"][cs(lw)]
    inter = orc.attention_interior(cfg, q.reshape(s, b, lw), k.reshape(s, b, lw), rank * lh, lh)
    sm, mk, sd = inter
    o = np.zeros((s, b, lw))
    V = v.reshape(s, b, lw)
    for hh in range(lh):
        for j in range(b):
            o[:, j, hh * hd:(hh + 1) * hd] = sd[hh, j] @ V[:, j, hh * hd:(hh + 1) * hd]
    O = o.reshape(s * b, lw)
    a = rs(O @ W["wo"][cs(lw), :]) + W["bo"]
    am = mask(1)
    r1 = xs + a * am * inv
    y2, mu2, iv2 = ln(r1, W["ln2_gain"], W["ln2_bias"])
    Y2 = ag(y2)
    gin = Y2 @ W["w1"][:, cs(fw)] + W["b1"][cs(fw)]
    fin = gelu(gin)
    m = rs(fin @ W["w2"][cs(fw), :]) + W["b2"]
    mm = mask(2)
    y = r1 + m * mm * inv
    # backward (block.cpp:642-726)
    dys = dy.reshape(s * b, h)[rank * RL:(rank + 1) * RL]
    dmo = dys * mm * inv
    db2 = dmo.sum(0)
    DMO = ag(dmo)
    Y2b = ag(y2)
    dgin = (DMO @ W["w2"][cs(fw), :].T) * dgelu(gin)
    dy2 = rs(dgin @ W["w1"][:, cs(fw)].T)
    dx2, dg2, dbe2 = ln_bwd(dy2, r1, mu2, iv2, W["ln2_gain"])
    dr1 = dys + dx2
    dao = dr1 * am * inv
    dbo = dao.sum(0)
    DAO = ag(dao)
    dO = (DAO @ W["wo"][cs(lw), :].T).reshape(s, b, lw)
    dq = np.zeros((s, b, lw)); dk = np.zeros_like(dq); dv = np.zeros_like(dq)
    Q, K = q.reshape(s, b, lw), k.reshape(s, b, lw)
    sc = 1 / np.sqrt(hd)
    for hh in range(lh):
        for j in range(b):
            sl = slice(hh * hd, (hh + 1) * hd)
            dsd = dO[:, j, sl] @ V[:, j, sl].T
            dv[:, j, sl] = sd[hh, j].T @ dO[:, j, sl]
            dsm = dsd * mk[hh, j] * inv
            rowdot = (dsm * sm[hh, j]).sum(1, keepdims=True)
            dsc = sm[hh, j] * (dsm - rowdot)
            dq[:, j, sl] = dsc @ K[:, j, sl] * sc
            dk[:, j, sl] = dsc.T @ Q[:, j, sl] * sc
    dY1 = (dq.reshape(s * b, lw) @ W["wq"][:, cs(lw)].T + dk.reshape(s * b, lw) @ W["wk"][:, cs(lw)].T
           + dv.reshape(s * b, lw) @ W["wv"][:, cs(lw)].T)
    dy1 = rs(dY1)
    dx1, dg1, dbe1 = ln_bwd(dy1, xs, mu1, iv1, W["ln1_gain"])
    dx = dr1 + dx1
    repl = torch.from_numpy(np.concatenate([dbo, db2, dg1, dbe1, dg2, dbe2]))
    dist.all_reduce(repl)  # the six GradSync all-reduces, packed
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), y=y, dx=dx, repl=repl.numpy(),
             w1=(Y2b.T @ dgin))


@pytest.mark.parametrize("world", [2])
def test_rank_program_matches_simulated_ranks(tmp_path, world, orc):
    _run(world, _seqpar_rank_program, str(tmp_path))
    cfg = orc.BlockConfig(heads=4, hidden=16, seq=8, batch=2, dropout_p=0.1, seed=42)
    x = orc.random_uniform(orc.hash_counter(42, 1000), (8, 2, 16), -1, 1)
    dy = orc.random_uniform(orc.hash_counter(42, 2000), (8, 2, 16), -1, 1)
    P = orc.params_random(16, orc.hash_counter(42, 3000))
    ref = orc.seqpar_layer(cfg, world, P, x, dy)
    G = orc.unpack(16, ref.grads)
    R = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    y = np.concatenate([r["y"] for r in R]).reshape(8, 2, 16)
    dx = np.concatenate([r["dx"] for r in R]).reshape(8, 2, 16)
    assert np.max(np.abs(y - ref.y)) <= 1e-10
    assert np.max(np.abs(dx - ref.dx)) <= 1e-10
    repl = np.concatenate([G[n] for n in ("bo", "b2", "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias")])
    for r in R:
        assert np.max(np.abs(r["repl"] - repl)) <= 1e-10
    for i, r in enumerate(R):
        assert np.max(np.abs(r["w1"] - ref.w1_grad_shards[i])) <= 1e-10
