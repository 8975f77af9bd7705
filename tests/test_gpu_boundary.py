"""The free-standing reference functions through the C ABI on the GPU, against the reference:
  attention_interior(q, k, cfg, head_offset, local_heads)  block.cpp:381-417
  all_gather / reduce_scatter / all_reduce (fp64)          collectives.cpp:21-73
  reference_block_forward / _backward                      block.cpp:419-510
  seqpar_block_forward(RankShardedTensor)                  block.hpp:158-162
Masks, fp64 collectives and CommLog counters bit-exact (the reference sums partials in rank
order, the device kernel too); f32 interiors within 1e-6; bf16 within 1e-2.
"""
import numpy as np
import pytest

import golden_layer as G
from test_gpu_layer import spl  # noqa: F401

pytestmark = pytest.mark.gpu


def _ref():
    from oracle import ref as R
    return R if R.available() else None


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape,offs", [
    (dict(heads=2, hidden=8, seq=4, batch=1), [(0, 2), (1, 1)]),
    (dict(heads=8, hidden=64, seq=32, batch=2), [(0, 8), (2, 2), (6, 2), (4, 4)]),
    (dict(heads=4, hidden=512, seq=256, batch=2), [(0, 4), (2, 2)]),
])
@pytest.mark.parametrize("causal", [False, True])
def test_attention_interior_vs_oracle(spl, orc, dtype, shape, offs, causal):
    cfg = orc.BlockConfig(**shape, dropout_p=0.1, causal=causal)
    scfg = spl.BlockConfig(cfg.heads, cfg.hidden, cfg.seq, cfg.batch, 0.1, causal, 42)
    R = _ref()
    hd = cfg.hidden // cfg.heads
    for off, lh in offs:
        q = orc.random_uniform(11 + off, (cfg.seq, cfg.batch, lh * hd), -1, 1)
        k = orc.random_uniform(12 + off, (cfg.seq, cfg.batch, lh * hd), -1, 1)
        if dtype == "bf16":  # compare on the bf16-rounded operands the kernel sees
            import torch
            q = torch.from_numpy(q).bfloat16().double().numpy()
            k = torch.from_numpy(k).bfloat16().double().numpy()
        got = spl.attention_interior(q, k, scfg, off, lh, dtype=dtype)
        want = orc.attention_interior(cfg, q, k, off, lh)
        assert np.array_equal(got[1], want[1])
        tol = 1e-6 if dtype == "f32" else 1e-2
        assert np.max(np.abs(got[0] - want[0])) <= tol
        assert np.max(np.abs(got[2] - want[2])) <= tol / 0.9
        if R is not None:
            assert np.array_equal(R.attention_interior(cfg, q, k, off, lh)[1], got[1])


def test_attention_interior_errors(spl):
    cfg = spl.BlockConfig(8, 64, 32, 2, 0.1, False, 42)
    q = np.zeros((32, 2, 16))
    with pytest.raises(ValueError):
        spl.attention_interior(q, q, cfg, 1, 2)  # offset not a multiple of local_heads
    with pytest.raises(ValueError):
        spl.attention_interior(q, q, cfg, 0, 3)  # heads % local_heads != 0
    with pytest.raises(ValueError):
        spl.attention_interior(np.zeros((32, 2, 8)), q, cfg, 0, 2)


@pytest.mark.parametrize("t", [1, 2, 3, 4, 8])
def test_collectives_fp64_bit_exact(spl, t):
    rs = np.random.default_rng(t)
    parts = [rs.standard_normal((8, 3, 5)) for _ in range(t)]
    R = _ref()
    acc = parts[0].copy()
    for p in parts[1:]:
        acc = acc + p  # ordered_sum (collectives.cpp:30-38)
    for axis in range(3):
        full, log = spl.all_gather(parts, axis)
        assert np.array_equal(full, np.concatenate(parts, axis))
        assert log["schedule"]["all_gathers"] == 1
        assert log["schedule"]["ring_elements"] == (full.size // t) * (t - 1)
        if parts[0].shape[axis] % t == 0:
            sc, log = spl.reduce_scatter(parts, axis, tag="regather")
            assert all(np.array_equal(a, b) for a, b in zip(sc, np.split(acc, t, axis)))
            assert log["regather"]["reduce_scatters"] == 1
            if R is not None:
                want, rlog = R.reduce_scatter(np.stack(parts), axis, tag=1)
                assert all(np.array_equal(a, b) for a, b in zip(sc, want))
                assert rlog.regather.ring_elements == log["regather"]["ring_elements"]
        else:
            with pytest.raises(ValueError):
                spl.reduce_scatter(parts, axis)
    tot, log = spl.all_reduce(parts, tag="grad_sync")
    assert np.array_equal(tot, acc)
    assert log["grad_sync"]["ring_elements"] == 2 * (acc.size // t) * (t - 1)
    if R is not None:
        want, _ = R.all_reduce(np.stack(parts))
        assert np.array_equal(tot, want)


def test_collectives_reject_ragged(spl):
    ragged = [np.zeros((2, 2)), np.zeros((2, 3))]
    for fn in (lambda: spl.all_reduce(ragged), lambda: spl.all_gather(ragged, 0),
               lambda: spl.reduce_scatter(ragged, 0)):
        with pytest.raises(ValueError):
            fn()
    with pytest.raises(ValueError):
        spl.all_gather([], 0)


def test_reference_block_vs_golden(spl, orc):
    """reference_block_forward/backward at the toy golden shape (t = 1 fixtures of the
    reference's own block.cpp), and bit-identity with seqpar at t = 1 (test_seqpar.cpp:161-168)."""
    for case in [c for c in G.cases("toy") if c.t == 1]:
        cfg = case.cfg(orc)
        x, dy, p = case.inputs(orc)
        scfg = spl.BlockConfig(cfg.heads, cfg.hidden, cfg.seq, cfg.batch, cfg.dropout_p, cfg.causal, 42)
        fwd = spl.reference_block_forward(x, p, scfg)
        g = spl.reference_block_backward(dy, fwd, p)
        y_ref = case.get("y")
        assert np.max(np.abs(fwd.y - y_ref)) <= 1e-5 * np.max(np.abs(y_ref))
        assert np.linalg.norm(g.dx - case.get("dx")) <= 1e-4 * np.linalg.norm(case.get("dx"))
        sf = spl.seqpar_block_forward([x], p, 1, scfg)
        assert np.array_equal(sf.y_shards[0], fwd.y)
        assert sum(v[1] for v in fwd.ledger.values()) == 1248  # test_seqpar.cpp:120-137
        m = fwd.saved("attn_dropout_mask")
        assert m.size == 32 and set(np.unique(m)) <= {0.0, 1.0}


def test_sharded_overload_and_param_reload(spl, orc):
    cfg = orc.BlockConfig(heads=8, hidden=64, seq=32, batch=2, dropout_p=0.1)
    scfg = spl.BlockConfig(8, 64, 32, 2, 0.1, False, 42)
    x = orc.random_uniform(5, (32, 2, 64), -1, 1)
    dy = orc.random_uniform(6, (32, 2, 64), -1, 1)
    p1 = orc.params_random(64, 7)
    p2 = orc.params_random(64, 8)
    a = spl.seqpar_block_forward_sharded(spl.RankShardedTensor.from_full(x, "sequence", 0, 4), p1, scfg)
    b = spl.seqpar_block_forward(np.split(x, 4, 0), p1, 4, scfg)
    assert a.t == 4 and all(np.array_equal(u, v) for u, v in zip(a.y_shards, b.y_shards))
    with pytest.raises(ValueError):
        spl.seqpar_block_forward_sharded(spl.RankShardedTensor.from_full(x, "hidden", 2, 4), p1, scfg)
    # backward with other params: the backward GEMMs use them (block.cpp:639-640) — the
    # result differs from the same-param backward, and the forward's y is unaffected
    g1 = spl.seqpar_block_backward(np.split(dy, 4, 0), a, p1)
    c = spl.seqpar_block_forward(np.split(x, 4, 0), p1, 4, scfg)
    g2 = spl.seqpar_block_backward(np.split(dy, 4, 0), c, p2)
    assert not np.allclose(np.concatenate(g1.dx_shards), np.concatenate(g2.dx_shards))
    # with recompute="full" the combination is rejected
    f = spl.seqpar_block_forward(np.split(x, 4, 0), p1, 4, scfg, recompute="full")
    with pytest.raises(ValueError):
        spl.seqpar_block_backward(np.split(dy, 4, 0), f, p2)
