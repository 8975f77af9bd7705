"""GPU tests of the microbatch window executor (spl_window_*).

  * numerics: every microbatch of a windowed 1F1B run gives bit-for-bit the y / dx of a
    standalone stack of its mode (no recompute when fully stored, the inner regime when
    checkpointed) with MaskKey microbatch i, and the window's parameter gradients are bit-for-bit
    the running fp32 sum of the standalone gradients in backward order;
  * memory: the peak ledger bytes of live microbatches equals the per-rank peak of
    simulate_memory_with_modes (pipeline_sim.cpp:222-275) for the plan's modes, and every slot
    stays within the plan's budget.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPE = dict(heads=4, hidden=256, seq=128, batch=2)


@pytest.fixture(scope="module")
def spl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2205_05198_b200 as m
    return m


def _inputs(torch, n_mb, local, shp, seed):
    g = torch.Generator(device="cuda:0").manual_seed(seed)
    mk = lambda: [(torch.rand(shp, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa
                  for _ in range(local)]
    return [mk() for _ in range(n_mb)], [mk() for _ in range(n_mb)]


# the last case is large enough for the fused all-gather (h/t >= 256, RF multiple of 256)
WIDE = dict(heads=8, hidden=1024, seq=256, batch=2)


@pytest.mark.parametrize("inner,t,p,stage,modes,shape", [
    ("selective", 1, 3, 0, [1, 0, 0, 1, 0], SHAPE),
    ("full", 2, 3, 1, [0, 1, 1, 0], SHAPE),
    ("selective", 2, 2, 0, [0, 0, 0], SHAPE),
    ("full", 1, 2, 1, [1, 1, 1], SHAPE),
    ("selective", 2, 2, 0, [1, 0, 1], WIDE),
])
def test_window_matches_standalone(spl, inner, t, p, stage, modes, shape):
    import torch
    L = 2
    cfg = spl.BlockConfig(**shape, dropout_p=0.1, seed=42)
    w = spl.SeqparWindow(cfg, t, L, p, stage, modes, recompute=inner)
    for l, lay in enumerate(w.layers):
        lay.init_params(100 + l)
    shp = w.shard_shape()
    x, dy = _inputs(torch, len(modes), w.local, shp, 7)
    y, dx = w.run(x, dy)
    torch.cuda.synchronize()
    got = [lay.grads() for lay in w.layers]
    acc = [None] * L
    for i, m in enumerate(modes):  # backward order of the rank program: microbatch 1..n_mb
        ci = spl.BlockConfig(**shape, dropout_p=0.1, seed=42, microbatch=i + 1)
        st = spl.SeqparStack(ci, t, L, "none" if m else inner, check_finite=False)
        for l, lay in enumerate(st.layers):
            lay.init_params(100 + l)
        yi = st.forward(x[i])
        dxi = st.backward(dy[i])
        torch.cuda.synchronize()
        for r in range(w.local):
            assert torch.equal(yi[r], y[i][r]), (i, r)
            assert torch.equal(dxi[r], dx[i][r]), (i, r)
        for l, lay in enumerate(st.layers):
            gi = lay.grads().astype(np.float32)
            acc[l] = gi if acc[l] is None else (acc[l] + gi).astype(np.float32)
        st.close()
    for l in range(L):
        np.testing.assert_array_equal(got[l].astype(np.float32), acc[l])
    w.close()


@pytest.mark.parametrize("inner,seq", [("selective", 512), ("full", 128)])
def test_window_memory_matches_plan(spl, inner, seq):
    import torch
    L, p, stage, n_mb = 2, 4, 1, 6
    shape = {**SHAPE, "seq": seq}  # selective: s large enough that the interior dominates
    m = spl.ModelShape(heads=shape["heads"], hidden=shape["hidden"], layers=L * p,
                       seq=seq, vocab=16, tensor=1, pipeline=p,
                       microbatch=shape["batch"], microbatches=n_mb, recompute=inner)
    full, ckpt = spl.microbatch_bytes(m, stage)  # stage > 0: no embedding / output extras
    lo = spl.window_plan(m, 2**63 - 1)["min_feasible_budget"]  # stage 0's 4 slots
    budget = max(full + 2 * ckpt, lo)  # one fully stored microbatch beside two checkpointed
    plan = spl.window_plan(m, budget)
    row = plan["modes"][stage]
    assert 0 < sum(row) < n_mb
    _, peak = spl.stage_timeline(m, stage, row, True)
    cfg = spl.BlockConfig(**shape, dropout_p=0.1, seed=42)
    w = spl.SeqparWindow(cfg, 1, L, p, stage, row, recompute=inner)
    w.init_params(5)
    x, dy = _inputs(torch, n_mb, w.local, w.shard_shape(), 3)
    w.run(x, dy)
    torch.cuda.synchronize()
    mem = w.memory()
    assert mem["live_peak_ledger"] == peak <= budget
    assert mem["slots_ledger"] == mem["fully_stored_slots"] * full + mem["checkpointed_slots"] * ckpt
    w.close()


def test_window_errors(spl):
    cfg = spl.BlockConfig(**SHAPE, dropout_p=0.1, seed=42)
    with pytest.raises(ValueError):
        spl.SeqparWindow(cfg, 1, 1, 3, 0, [1, 0])  # n_mb < p
    with pytest.raises(ValueError):
        spl.SeqparWindow(cfg, 1, 1, 2, 0, [1, 0], recompute="none")  # checkpointed needs inner
    with pytest.raises(ValueError):
        spl.SeqparWindow(cfg, 1, 1, 2, 2, [1, 0])  # stage >= p


def test_window_f32_accumulation(spl):
    """The exact-fp32 execution dtype (SIMT GEMMs): accumulated gradients equal the fp32 running
    sum of standalone runs bit-for-bit (the SIMT epilogue's C += A·B path)."""
    import torch
    L, t, p, stage, modes = 1, 2, 2, 0, [1, 0, 0]
    cfg = spl.BlockConfig(**SHAPE, dropout_p=0.1, seed=42)
    w = spl.SeqparWindow(cfg, t, L, p, stage, modes, recompute="selective", dtype="f32")
    w.layers[0].init_params(3)
    g = torch.Generator(device="cuda:0").manual_seed(5)
    shp = w.shard_shape()
    mk = lambda: [(torch.rand(shp, generator=g, device="cuda") * 2 - 1) for _ in range(t)]  # noqa
    x = [mk() for _ in modes]
    dy = [mk() for _ in modes]
    y, dx = w.run(x, dy)
    torch.cuda.synchronize()
    got = w.layers[0].grads()
    acc = None
    for i, m in enumerate(modes):
        ci = spl.BlockConfig(**SHAPE, dropout_p=0.1, seed=42, microbatch=i + 1)
        st = spl.SeqparStack(ci, t, L, "none" if m else "selective", dtype="f32", check_finite=False)
        st.layers[0].init_params(3)
        yi = st.forward(x[i])
        dxi = st.backward(dy[i])
        torch.cuda.synchronize()
        for r in range(t):
            assert torch.equal(yi[r], y[i][r]) and torch.equal(dxi[r], dx[i][r])
        gi = st.layers[0].grads().astype(np.float32)
        acc = gi if acc is None else (acc + gi).astype(np.float32)
        st.close()
    np.testing.assert_array_equal(got.astype(np.float32), acc)
    w.close()
