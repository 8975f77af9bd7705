"""GPU parity of the B200 layer (libspl.so through the C ABI) against the fp64 oracle.

Tolerances (stated here as the contract):
  masks, ledger bytes ........................ bit-exact
  fp32 path: y max-abs <= 1e-5 * max|y_ref|; dx and param grads rel-L2 <= 1e-4
  bf16 path: y, dx rel-L2 <= 1e-2; weight grads rel-L2 <= 2e-2
Mirrors the reference suites test_seqpar.cpp:120-271 and verify.cpp:107-321.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TINY = dict(heads=8, hidden=256, seq=128, batch=2)  # BASELINE configs[0]


@pytest.fixture(scope="module")
def spl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2205_05198_b200 as m
    return m


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def make_case(orc, shape, seed=42, dropout=0.1, causal=False, key=0):
    cfg = orc.BlockConfig(**shape, dropout_p=dropout, causal=causal, seed=seed)
    shp = (cfg.seq, cfg.batch, cfg.hidden)
    x = orc.random_uniform(orc.hash_counter(seed, 1000 + key), shp, -1, 1)
    dy = orc.random_uniform(orc.hash_counter(seed, 2000 + key), shp, -1, 1)
    p = orc.params_random(cfg.hidden, orc.hash_counter(seed, 3000 + key))
    return cfg, x, dy, p


def to_spl_cfg(spl, cfg):
    return spl.BlockConfig(cfg.heads, cfg.hidden, cfg.seq, cfg.batch, cfg.dropout_p, cfg.causal,
                           cfg.seed, cfg.layer_index, cfg.microbatch, cfg.layer_norm_eps)


def run(spl, cfg, t, p, x, dy, recompute="none", sp=True, dtype="f32"):
    import torch
    c = to_spl_cfg(spl, cfg)
    L = spl.SeqparLayer(c, t, recompute, sp, dtype)
    L.load_params(p)
    td = torch.float32 if dtype == "f32" else torch.bfloat16
    if sp:
        xs = [torch.from_numpy(s.copy()).to("cuda", td) for s in np.split(x, t, axis=0)]
        ds = [torch.from_numpy(s.copy()).to("cuda", td) for s in np.split(dy, t, axis=0)]
    else:
        xs = [torch.from_numpy(x).to("cuda", td) for _ in range(t)]
        ds = [torch.from_numpy(dy).to("cuda", td) for _ in range(t)]
    y = L.forward(xs)
    dx = L.backward(ds)
    cat = (lambda v: np.concatenate([u.double().cpu().numpy() for u in v], 0)) if sp else \
          (lambda v: v[0].double().cpu().numpy())
    return L, cat(y), cat(dx), L.grads()


def grads_close(orc, h, got, want, tol):
    """Per-tensor rel-L2, the denominator floored at 3% of a global-RMS-sized tensor, so
    tensors whose exact gradient is ~0 (the key bias: softmax is shift-invariant, its fp64
    gradient is 1e-15) compare on the layer's gradient scale instead of on rounding noise."""
    G, R = orc.unpack(h, got), orc.unpack(h, want)
    rms = float(np.sqrt(np.mean(want ** 2)))
    for name in G:
        err = np.linalg.norm(G[name] - R[name])
        assert err <= tol * (np.linalg.norm(R[name]) + 0.03 * rms * np.sqrt(R[name].size)), (name, err)


def check_f32(spl, orc, res, ref, p):
    L, y, dx, g = res
    assert np.max(np.abs(y - ref.y)) <= 1e-5 * np.max(np.abs(ref.y))
    assert rel_l2(dx, ref.dx) <= 1e-4
    grads_close(orc, L.cfg.hidden, g, ref.grads, 1e-4)


@pytest.mark.parametrize("t", [1, 2, 4])
@pytest.mark.parametrize("recompute", ["none", "selective", "full"])
def test_tiny_f32_parity(spl, orc, t, recompute):
    cfg, x, dy, p = make_case(orc, TINY)
    ref = orc.seqpar_layer(cfg, t, p, x, dy)
    res = run(spl, cfg, t, p, x, dy, recompute)
    check_f32(spl, orc, res, ref, p)


@pytest.mark.parametrize("sp", [True, False])
def test_tiny_f32_causal_and_sp_off(spl, orc, sp):
    cfg, x, dy, p = make_case(orc, TINY, causal=True, key=1)
    ref = orc.seqpar_layer(cfg, 2, p, x, dy)
    res = run(spl, cfg, 2, p, x, dy, "selective", sp=sp)
    check_f32(spl, orc, res, ref, p)


def test_toy_shapes_f32(spl, orc):
    """verify.cpp:107-147 style: random toy shapes (unaligned widths) at t in {1,2,4}."""
    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0])
    from test_oracle_layer import CaseRng, random_toy_config
    seed = 42
    rng = CaseRng(orc, orc.hash_counter(seed, 2))
    n = 0
    for shape_idx in range(8):
        cfg = random_toy_config(orc, rng, seed, shape_idx)
        cfg.dropout_p = 0.1
        shp = (cfg.seq, cfg.batch, cfg.hidden)
        x = orc.random_uniform(orc.hash_counter(seed, 1000 + shape_idx), shp, -1, 1)
        lw = orc.random_uniform(orc.hash_counter(seed, 2000 + shape_idx), shp, -1, 1)
        p = orc.params_random(cfg.hidden, orc.hash_counter(seed, 3000 + shape_idx))
        for t in (1, 2, 4):
            if cfg.heads % t or cfg.seq % t:
                continue
            ref = orc.seqpar_layer(cfg, t, p, x, lw)
            for rc in ("none", "selective"):
                L, y, dx, g = run(spl, cfg, t, p, x, lw, rc)
                assert np.max(np.abs(y - ref.y)) <= 1e-5 * np.max(np.abs(ref.y))
                assert np.max(np.abs(dx - ref.dx)) <= 1e-4 * max(1.0, np.max(np.abs(ref.dx)))
                assert np.max(np.abs(g - ref.grads)) <= 1e-4 * max(1.0, np.max(np.abs(ref.grads)))
                n += 1
    assert n >= 8


@pytest.mark.parametrize("t,recompute", [(1, "none"), (1, "selective"), (2, "selective"), (2, "full")])
def test_tiny_bf16_parity(spl, orc, t, recompute):
    cfg, x, dy, p = make_case(orc, TINY)
    ref = orc.seqpar_layer(cfg, t, p, x, dy)
    L, y, dx, g = run(spl, cfg, t, p, x, dy, recompute, dtype="bf16")
    assert rel_l2(y, ref.y) <= 1e-2
    assert rel_l2(dx, ref.dx) <= 1e-2
    grads_close(orc, cfg.hidden, g, ref.grads, 2e-2)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_masks_bit_exact(spl, orc, dtype):
    cfg, x, dy, p = make_case(orc, TINY, key=2)
    t = 2
    ref = orc.seqpar_layer(cfg, t, p, x, dy, want_interior=True)
    L, *_ = run(spl, cfg, t, p, x, dy, "none", dtype=dtype)
    s, b, h, a = cfg.seq, cfg.batch, cfg.hidden, cfg.heads
    for op, name in ((1, "attn_dropout_mask"), (2, "mlp_dropout_mask")):
        key = orc.mask_key_fold(cfg.seed, 0, op, 1)
        full = orc.dropout_mask(key, s * b * h, cfg.dropout_p).reshape(s, b, h)
        for r in range(t):
            got = L.saved(r, name, (s // t, b, h))
            assert np.array_equal(got, full[r * s // t:(r + 1) * s // t])
    lh = a // t
    for r in range(t):
        got = L.saved(r, "softmax_dropout_mask", (lh, b, s, s))
        assert np.array_equal(got, ref.interior[1][r * lh:(r + 1) * lh])


@pytest.mark.parametrize("side", ["keep", "drop"])
def test_keep_bits_threshold_tie(spl, orc, side):
    """The keep-bit pass decides a key on the high word of its hash and re-derives a word when a
    high word equals the threshold's (probability 2^-32 per key): pick p so that key 0 of the
    softmax-dropout mask ties, with the low word on either side of the threshold."""
    import dataclasses
    # head_dim 64: the tcgen05 attention, which reads the keep-bit pass's bits
    cfg, x, dy, p = make_case(orc, dict(heads=4, hidden=256, seq=128, batch=2), key=5)
    key = orc.mask_key_fold(cfg.seed, 0, 0, 1)  # softmax dropout (rng.cuh kSoftmaxDrop)
    h = orc.hash_counter(key, 0)
    lo = h & 0xffffffff
    r = (lo >> 11) if side == "keep" else (lo >> 11) + 1  # threshold low word r<<11 vs lo
    assert r < (1 << 21)
    T = ((h >> 32) << 21) | r  # keep iff h >= T * 2^11 (rng.cpp:35-37, block.cpp:63)
    ptie = T / float(2**53)
    assert int(np.ceil(ptie * 2.0**53)) == T and 0 < ptie < 1
    cfg = dataclasses.replace(cfg, dropout_p=ptie)
    L, *_ = run(spl, cfg, 1, p, x, dy, "none", dtype="bf16")
    s, b, a = cfg.seq, cfg.batch, cfg.heads
    got = L.saved(0, "softmax_dropout_mask", (a, b, s, s))
    want = orc.dropout_mask(key, a * b * s * s, ptie).reshape(a, b, s, s)
    assert want[0, 0, 0, 0] == (1.0 if side == "keep" else 0.0)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_recompute_bit_exact(spl, orc, dtype):
    """test_seqpar.cpp:248-271 on the device: the interior recomputed from the stored Q/K by
    the kernel equals the stored one bit-for-bit; 5as²b/t bytes are discarded by selective."""
    cfg, x, dy, p = make_case(orc, TINY, key=3)
    t = 2
    L, *_ = run(spl, cfg, t, p, x, dy, "none", dtype=dtype)
    s, b, a = cfg.seq, cfg.batch, cfg.heads
    lh = a // t
    for r in range(t):
        redone = L.interior(r)
        for i, name in enumerate(("softmax_out", "softmax_dropout_mask", "softmax_dropout_out")):
            assert np.array_equal(redone[i], L.saved(r, name, (lh, b, s, s)))
    sel = spl.SeqparLayer(to_spl_cfg(spl, cfg), t, "selective", True, dtype)
    none_l = sum(v[1] for v in L.ledger(0).values())
    sel_l = sum(v[1] for v in sel.ledger(0).values())
    assert none_l - sel_l == 5 * a * s * s * b // t


def test_interior_matches_oracle(spl, orc):
    cfg, x, dy, p = make_case(orc, TINY, key=4, causal=True)
    ref = orc.seqpar_layer(cfg, 2, p, x, dy, want_interior=True)
    L, *_ = run(spl, cfg, 2, p, x, dy, "selective")
    lh = cfg.heads // 2
    for r in range(2):
        got = L.interior(r)
        assert np.array_equal(got[1], ref.interior[1][r * lh:(r + 1) * lh])
        assert np.max(np.abs(got[0] - ref.interior[0][r * lh:(r + 1) * lh])) <= 1e-5
        assert np.max(np.abs(got[2] - ref.interior[2][r * lh:(r + 1) * lh])) <= 2e-5


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_device_init_equals_host_params(spl, orc, dtype):
    import torch
    cfg, x, dy, _ = make_case(orc, TINY, key=5)
    c = to_spl_cfg(spl, cfg)
    A = spl.SeqparLayer(c, 2, "selective", True, dtype)
    B = spl.SeqparLayer(c, 2, "selective", True, dtype)
    A.init_params(1234)
    B.load_params(orc.params_random(cfg.hidden, 1234))
    td = torch.float32 if dtype == "f32" else torch.bfloat16
    xs = [torch.from_numpy(s.copy()).to("cuda", td) for s in np.split(x, 2, 0)]
    ya, yb = A.forward(xs), B.forward(xs)
    for u, v in zip(ya, yb):
        assert torch.equal(u, v)


@pytest.mark.parametrize("recompute", ["none", "selective", "full"])
@pytest.mark.parametrize("sp", [True, False])
@pytest.mark.parametrize("t", [1, 2, 4])
def test_ledger_equals_accountant(spl, orc, recompute, sp, t):
    cfg, x, dy, p = make_case(orc, TINY)
    L = spl.SeqparLayer(to_spl_cfg(spl, cfg), t, recompute, sp, "bf16")
    led, phys, unc = L.saved_bytes(0)
    acc = orc.per_layer_bytes(cfg.heads, cfg.hidden, cfg.seq, cfg.batch, t, recompute, sp)
    if recompute == "full" and sp:
        # reference convention counts A·sbh for full recompute regardless of t/SP
        # (activation_memory.cpp:59-63); the device holds only the x shard, sbh/t.
        assert led * t == acc
    else:
        assert led == acc
    assert phys == led  # bf16 = 2 bytes, masks 1 byte: physical equals the convention


def test_comm_log_counts(spl, orc):
    cfg, x, dy, p = make_case(orc, TINY)
    L, *_ = run(spl, cfg, 2, p, x, dy, "selective")
    c = L.comm_log()
    assert c["schedule"]["all_gathers"] == 4 and c["schedule"]["reduce_scatters"] == 4
    assert c["schedule"]["all_reduces"] == 0
    assert c["regather"]["all_gathers"] == 2 and c["grad_sync"]["all_reduces"] == 6
    assert c["schedule"]["ring_elements"] * 2 == orc.layer_comm_bytes_sp(cfg.seq, cfg.batch, cfg.hidden, 2)
    assert c["schedule"]["ring_elements"] * 2 == spl.layer_comm_bytes(cfg.seq, cfg.batch, cfg.hidden, 2, 2, True)


def test_errors(spl, orc):
    import torch
    cfg, x, dy, p = make_case(orc, TINY)
    c = to_spl_cfg(spl, cfg)
    with pytest.raises(ValueError):
        spl.SeqparLayer(c, 3, "none", True, "f32")  # heads/seq not divisible
    L = spl.SeqparLayer(c, 2, "none", True, "f32")
    L.load_params(p)
    ds = [torch.zeros((64, 2, 256), device="cuda") for _ in range(2)]
    with pytest.raises(ValueError):  # missing saved forward state
        L.backward(ds)
    xs = [torch.from_numpy(s.copy()).to("cuda", torch.float32) for s in np.split(x, 2, 0)]
    xs[0][0, 0, 0] = float("inf")
    with pytest.raises(ArithmeticError):
        L.forward(xs)


def test_identity_like_block(spl, orc):
    """test_seqpar.cpp:234-246: zero weights -> dx == dy exactly, b2/bo grads = column sums."""
    import torch
    cfg = orc.BlockConfig(**TINY)
    dy = orc.random_uniform(61, (cfg.seq, cfg.batch, cfg.hidden), -1, 1)
    L = spl.SeqparLayer(to_spl_cfg(spl, cfg), 1, "none", True, "f32")
    L.load_params(orc.params_zeros(cfg.hidden))
    y = L.forward([torch.zeros((cfg.seq, cfg.batch, cfg.hidden), device="cuda")])
    assert torch.count_nonzero(y[0]).item() == 0
    d = torch.from_numpy(dy).to("cuda", torch.float32)
    dx = L.backward([d])
    assert torch.equal(dx[0], d)
    g = orc.unpack(cfg.hidden, L.grads())
    cs = d.double().reshape(-1, cfg.hidden).sum(0).cpu().numpy()
    assert np.max(np.abs(g["b2"] - cs)) <= 1e-4 and np.max(np.abs(g["bo"] - cs)) <= 1e-4


def test_facade_reference_api(spl, orc):
    """The reference-shaped functions (block.hpp:158-174) on the device."""
    cfg, x, dy, p = make_case(orc, TINY)
    c = to_spl_cfg(spl, cfg)
    fwd = spl.seqpar_block_forward(np.split(x, 2, 0), p, 2, c, "selective")
    back = spl.seqpar_block_backward(np.split(dy, 2, 0), fwd, p)
    ref = orc.seqpar_layer(cfg, 2, p, x, dy)
    assert np.max(np.abs(np.concatenate(fwd.y_shards) - ref.y)) <= 1e-5 * np.max(np.abs(ref.y))
    assert rel_l2(np.concatenate(back.dx_shards), ref.dx) <= 1e-4
    w1 = orc.unpack(cfg.hidden, ref.grads)["w1"]
    for r in range(2):
        assert rel_l2(back.w1_grad_shards[r], w1[:, r * 512:(r + 1) * 512]) <= 1e-4


@pytest.mark.parametrize("shape,t,causal", [
    (dict(heads=8, hidden=768, seq=256, batch=2), 1, False),    # head_dim 96 (22B)
    (dict(heads=8, hidden=1024, seq=192, batch=1), 2, True),    # head_dim 128 (175B), s tail
    (dict(heads=8, hidden=1280, seq=256, batch=1), 2, False),   # head_dim 160 (530B / 1T)
    (dict(heads=4, hidden=256, seq=160, batch=3), 1, True),     # head_dim 64, s tail
    # s % 128 == 0: the two-tile ping-pong forward (k_attention_fwd_pp.cu), causal diagonal
    # tiles in both query tiles and a CTA whose second tile is empty (s = 384)
    (dict(heads=4, hidden=512, seq=384, batch=1), 1, True),     # head_dim 128
    (dict(heads=8, hidden=512, seq=256, batch=2), 2, True),     # head_dim 64
])
@pytest.mark.parametrize("recompute", ["selective", "none"])
def test_bf16_head_dims(spl, orc, shape, t, causal, recompute):
    cfg, x, dy, p = make_case(orc, shape, causal=causal, key=7)
    ref = orc.seqpar_layer(cfg, t, p, x, dy)
    L, y, dx, g = run(spl, cfg, t, p, x, dy, recompute, dtype="bf16")
    assert rel_l2(y, ref.y) <= 1e-2
    assert rel_l2(dx, ref.dx) <= 1e-2
    grads_close(orc, cfg.hidden, g, ref.grads, 2e-2)


def test_nccl_rank_handle_matches_local(spl, orc):
    """One NCCL rank (t=1 group) runs the same schedule as the simulated-rank handle; this is
    the handle bench.py uses per GPU under torchrun (collectives become ncclAllGather /
    ncclReduceScatter / ncclAllReduce)."""
    import torch
    cfg, x, dy, p = make_case(orc, TINY)
    c = to_spl_cfg(spl, cfg)
    uid = spl.SeqparLayer.nccl_unique_id()
    A = spl.SeqparLayer(c, 1, "selective", True, "bf16", nccl=(0, uid))
    B = spl.SeqparLayer(c, 1, "selective", True, "bf16")
    for L in (A, B):
        L.load_params(p)
    xs = [torch.from_numpy(x).to("cuda", torch.bfloat16)]
    ds = [torch.from_numpy(dy).to("cuda", torch.bfloat16)]
    ya, yb = A.forward(xs), B.forward(xs)
    da, db = A.backward(ds), B.backward(ds)
    assert torch.equal(ya[0], yb[0]) and torch.equal(da[0], db[0])
    assert np.array_equal(A.grads(), B.grads())


@pytest.mark.parametrize("t,recompute", [(1, "selective"), (2, "selective"), (2, "full"), (2, "none")])
def test_cuda_graphs_bit_identical(spl, orc, t, recompute):
    """Forward/backward captured as CUDA graphs (multi-stream: comm + RNG streams joined by
    events) replay bit-identically to eager execution."""
    import torch
    cfg, x, dy, p = make_case(orc, dict(heads=8, hidden=512, seq=256, batch=2), key=9)
    c = to_spl_cfg(spl, cfg)
    outs = []
    for graphs in (False, True):
        L = spl.SeqparLayer(c, t, recompute, True, "bf16", check_finite=False)
        L.load_params(p)
        L.set_graphs(graphs)
        xs = [torch.from_numpy(s.copy()).to("cuda", torch.bfloat16) for s in np.split(x, t, 0)]
        ds = [torch.from_numpy(s.copy()).to("cuda", torch.bfloat16) for s in np.split(dy, t, 0)]
        ys = [torch.empty_like(v) for v in xs]
        dxs = [torch.empty_like(v) for v in xs]
        for _ in range(3):
            L.forward(xs, ys)
            L.backward(ds, dxs)
        torch.cuda.synchronize()
        outs.append(([v.clone() for v in ys], [v.clone() for v in dxs], L.grads(), L.launch_count()))
    (ye, de, ge, le), (yg, dg, gg, lg) = outs
    assert all(torch.equal(a, b) for a, b in zip(ye, yg))
    assert all(torch.equal(a, b) for a, b in zip(de, dg))
    assert np.array_equal(ge, gg)
    assert le == lg  # graph replays are counted like the eager launches


@pytest.mark.parametrize("t,pinned", [(1, True), (2, True), (1, False)])
def test_step_host_matches_device_step(spl, orc, t, pinned):
    """spl_step_host (the end-to-end path bench.py's e2e uses: H2D x/dy, fwd, bwd, D2H y/dx,
    copies overlapped with compute on a copy stream) equals the device-buffer calls bit-for-bit,
    for pinned and pageable host buffers, over repeated steps."""
    import torch
    cfg, x, dy, p = make_case(orc, dict(heads=8, hidden=512, seq=256, batch=2), key=11)
    c = to_spl_cfg(spl, cfg)
    A = spl.SeqparLayer(c, t, "selective", True, "bf16", check_finite=False)
    B = spl.SeqparLayer(c, t, "selective", True, "bf16", check_finite=False)
    A.load_params(p)
    B.load_params(p)
    xs = [torch.from_numpy(s.copy()).to("cuda", torch.bfloat16) for s in np.split(x, t, 0)]
    ds = [torch.from_numpy(s.copy()).to("cuda", torch.bfloat16) for s in np.split(dy, t, 0)]
    hx, hdy = torch.cat(xs).cpu(), torch.cat(ds).cpu()
    hy, hdx = torch.empty_like(hx), torch.empty_like(hx)
    if pinned:
        hx, hdy, hy, hdx = hx.pin_memory(), hdy.pin_memory(), hy.pin_memory(), hdx.pin_memory()
    for _ in range(3):
        y = A.forward(xs)
        dx = A.backward(ds)
        B.step_host(hx, hdy, hy, hdx)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(y).cpu(), hy)
    assert torch.equal(torch.cat(dx).cpu(), hdx)
    assert np.array_equal(A.grads(), B.grads())


def test_step_host_async_pipelined(spl, orc):
    """Several spl_step_host_async calls in flight over two host buffer sets (the bench's e2e
    loop) give every step the same results as synchronous device calls."""
    import torch
    cfg, x, dy, p = make_case(orc, dict(heads=8, hidden=512, seq=256, batch=2), key=12)
    c = to_spl_cfg(spl, cfg)
    A = spl.SeqparLayer(c, 1, "selective", True, "bf16", check_finite=False)
    B = spl.SeqparLayer(c, 1, "selective", True, "bf16", check_finite=False)
    A.load_params(p)
    B.load_params(p)
    xs = [torch.from_numpy(x).to("cuda", torch.bfloat16)]
    ds = [torch.from_numpy(dy).to("cuda", torch.bfloat16)]
    y = A.forward(xs)[0].cpu()
    dx = A.backward(ds)[0].cpu()
    hx = [xs[0].cpu().pin_memory() for _ in range(2)]
    hdy = [ds[0].cpu().pin_memory() for _ in range(2)]
    hy = [torch.full_like(hx[0], float("nan")).pin_memory() for _ in range(2)]
    hdx = [torch.full_like(hx[0], float("nan")).pin_memory() for _ in range(2)]
    for i in range(5):
        B.step_host_async(hx[i & 1], hdy[i & 1], hy[i & 1], hdx[i & 1])
    B.step_host_wait()
    for j in range(2):
        assert torch.equal(hy[j], y) and torch.equal(hdx[j], dx)
    assert np.array_equal(A.grads(), B.grads())


@pytest.mark.parametrize("shape,t", [(dict(heads=32, hidden=3072, seq=256, batch=2), 8),    # head_dim 96
                                     (dict(heads=16, hidden=2560, seq=256, batch=1), 8)])   # head_dim 160
def test_full_width_self_consistency(spl, orc, shape, t):
    """SURVEY.md §8c for shapes beyond what the fp64 oracle runs in seconds: the same layer on t
    simulated ranks (SP) equals the one-rank layer (same seed, masks identical by construction),
    and the three recompute regimes agree, within the bf16 tolerances."""
    import torch
    cfg = orc.BlockConfig(**shape, dropout_p=0.1, seed=42)
    c = to_spl_cfg(spl, cfg)
    shp = (cfg.seq, cfg.batch, cfg.hidden)
    g = torch.Generator().manual_seed(5)
    x = (torch.rand(shp, generator=g) * 2 - 1).to(torch.bfloat16)
    dy = (torch.rand(shp, generator=g) * 2 - 1).to(torch.bfloat16)
    res = {}
    for tt, rc in ((1, "selective"), (t, "selective"), (t, "none"), (t, "full")):
        L = spl.SeqparLayer(c, tt, rc, True, "bf16", check_finite=False)
        L.init_params(77)
        xs = [u.contiguous().cuda() for u in torch.chunk(x, tt, 0)]
        ds = [u.contiguous().cuda() for u in torch.chunk(dy, tt, 0)]
        y = torch.cat(L.forward(xs)).float().cpu()
        dx = torch.cat(L.backward(ds)).float().cpu()
        res[(tt, rc)] = (y.numpy(), dx.numpy(), L.grads())
        L.close()
    ref = res[(1, "selective")]
    for key, (y, dx, gr) in res.items():
        assert rel_l2(y, ref[0]) <= 1e-2, key
        assert rel_l2(dx, ref[1]) <= 1e-2, key
        assert rel_l2(gr, ref[2]) <= 2e-2, key


def test_spl_create_survey_form(spl, orc):
    """spl_create(desc, devices, t): t ranks on one device equal
    spl_create_local bit-for-bit; devices naming two GPUs are refused (one process per GPU)."""
    import ctypes as C
    import torch
    from paper_2205_05198_b200 import _lib
    from paper_2205_05198_b200.seqpar import _desc
    cfg, x, dy, p = make_case(orc, TINY, key=13)
    c = to_spl_cfg(spl, cfg)
    t = 2
    ref = spl.SeqparLayer(c, t, "selective", True, "bf16")
    ref.load_params(p)
    d = _desc(c, "selective", True, "bf16", True)
    h = C.c_void_p()
    devs = (C.c_int * t)(0, 0)
    _lib.check(_lib.lib().spl_create(C.byref(d), devs, t, C.byref(h)))
    L = spl.SeqparLayer(c, t, "selective", True, "bf16", _borrow=h)
    L.load_params(p)
    xs = [torch.from_numpy(s.copy()).to("cuda", torch.bfloat16) for s in np.split(x, t, 0)]
    ds = [torch.from_numpy(s.copy()).to("cuda", torch.bfloat16) for s in np.split(dy, t, 0)]
    for a, b in zip(ref.forward(xs), L.forward(xs)):
        assert torch.equal(a, b)
    for a, b in zip(ref.backward(ds), L.backward(ds)):
        assert torch.equal(a, b)
    np.testing.assert_array_equal(ref.grads(), L.grads())
    _lib.lib().spl_destroy(h)
    h2 = C.c_void_p()
    rc = _lib.lib().spl_create(C.byref(d), (C.c_int * 2)(0, 1), 2, C.byref(h2))
    assert rc == _lib.SPL_EINVAL


@pytest.mark.parametrize("causal", [False, True])
def test_bf16_no_dropout_tcgen05_attention(spl, orc, causal):
    """p = 0: the attention kernels run without keep bits (no keep-bit buffer is read); the
    two-tile ping-pong forward and the fused backward at head_dim 64, s % 128 == 0."""
    cfg, x, dy, p = make_case(orc, dict(heads=4, hidden=256, seq=256, batch=2), dropout=0.0,
                              causal=causal, key=11)
    ref = orc.seqpar_layer(cfg, 1, p, x, dy)
    L, y, dx, g = run(spl, cfg, 1, p, x, dy, "selective", dtype="bf16")
    assert rel_l2(y, ref.y) <= 1e-2
    assert rel_l2(dx, ref.dx) <= 1e-2
    grads_close(orc, cfg.hidden, g, ref.grads, 2e-2)
    L.close()


@pytest.mark.parametrize("causal", [False, True])
def test_bf16_stored_interior_vs_oracle(spl, orc, causal):
    """No-recompute regime, bf16, head_dim 64, s % 128 == 0: the stored interior written by the
    two-pass ping-pong forward (32-byte row stores) — softmax_out, the raw mask byte at every
    position (bit-exact) and softmax_dropout_out — against the oracle's interior."""
    shape = dict(heads=4, hidden=256, seq=256, batch=2)
    cfg, x, dy, p = make_case(orc, shape, causal=causal, key=12)
    ref = orc.seqpar_layer(cfg, 1, p, x, dy, want_interior=True)
    L, y, dx, g = run(spl, cfg, 1, p, x, dy, "none", dtype="bf16")
    n = ref.interior[0].size
    sm = L.saved(0, "softmax_out", (n,)).reshape(ref.interior[0].shape)
    mk = L.saved(0, "softmax_dropout_mask", (n,)).reshape(ref.interior[1].shape)
    sd = L.saved(0, "softmax_dropout_out", (n,)).reshape(ref.interior[2].shape)
    assert np.array_equal(mk, ref.interior[1])
    # bf16 storage: one rounding (2^-9 relative) of values <= 1 (P) and <= 1/(1-p) (P-tilde)
    assert np.max(np.abs(sm - ref.interior[0])) <= 4e-3
    assert np.max(np.abs(sd - ref.interior[2])) <= 5e-3
    assert rel_l2(y, ref.y) <= 1e-2
    L.close()
