"""GPU tests of the layer stack (spl_stack_*): L layers sharing one
workspace, each keeping only its own saved activations.

  * numerics: a 2-layer fp32 stack equals the oracle chain layer0 -> layer1 (layer_index 0, 1,
    so each layer draws its own masks; seqpar_block_forward/backward per layer, block.cpp:512-749)
    within the fp32 tolerances of test_gpu_layer.py; bf16 within the bf16 ones;
  * memory: Σ ledger over layers == total_first_stage_bytes(p = 1) bit-exactly
    (activation_memory.cpp:112-123) for none / selective (full: the device keeps the x shard,
    A·sbh/t per layer, the reference counts A·sbh); the shared workspace does not grow with L.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TINY = dict(heads=8, hidden=256, seq=128, batch=2)


@pytest.fixture(scope="module")
def spl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2205_05198_b200 as m
    return m


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _stack_case(orc, L, seed=42):
    shp = (TINY["seq"], TINY["batch"], TINY["hidden"])
    x = orc.random_uniform(orc.hash_counter(seed, 1000), shp, -1, 1)
    dy = orc.random_uniform(orc.hash_counter(seed, 2000), shp, -1, 1)
    ps = [orc.params_random(TINY["hidden"], orc.hash_counter(seed, 3000 + l)) for l in range(L)]
    return x, dy, ps


def _oracle_chain(orc, L, t, x, dy, ps):
    cfgs = [orc.BlockConfig(**TINY, dropout_p=0.1, seed=42, layer_index=l) for l in range(L)]
    acts = [x]
    for l in range(L - 1):
        acts.append(orc.seqpar_layer(cfgs[l], t, ps[l], acts[-1]).y)
    g, grads = dy, [None] * L
    y = None
    for l in reversed(range(L)):
        r = orc.seqpar_layer(cfgs[l], t, ps[l], acts[l], g)
        if l == L - 1:
            y = r.y
        g, grads[l] = r.dx, r.grads
    return y, g, grads


@pytest.mark.parametrize("dtype,recompute,t", [("f32", "selective", 1), ("f32", "none", 2),
                                               ("bf16", "selective", 2), ("bf16", "full", 1)])
def test_stack_matches_oracle_chain(spl, orc, dtype, recompute, t):
    import torch
    L = 2
    x, dy, ps = _stack_case(orc, L)
    y_ref, dx_ref, g_ref = _oracle_chain(orc, L, t, x, dy, ps)
    st = spl.SeqparStack(spl.BlockConfig(**TINY, dropout_p=0.1, seed=42), t, L, recompute, True, dtype)
    for l in range(L):
        st.layers[l].load_params(ps[l])
    td = torch.float32 if dtype == "f32" else torch.bfloat16
    xs = [torch.from_numpy(s.copy()).to("cuda", td) for s in np.split(x, t, axis=0)]
    ds = [torch.from_numpy(s.copy()).to("cuda", td) for s in np.split(dy, t, axis=0)]
    y = np.concatenate([u.double().cpu().numpy() for u in st.forward(xs)], 0)
    dx = np.concatenate([u.double().cpu().numpy() for u in st.backward(ds)], 0)
    if dtype == "f32":
        assert np.max(np.abs(y - y_ref)) <= 1e-5 * np.max(np.abs(y_ref))
        assert rel_l2(dx, dx_ref) <= 1e-4
        for l in range(L):
            assert rel_l2(st.layers[l].grads(), g_ref[l]) <= 1e-4
    else:
        assert rel_l2(y, y_ref) <= 1e-2
        assert rel_l2(dx, dx_ref) <= 1e-2
        for l in range(L):
            assert rel_l2(st.layers[l].grads(), g_ref[l]) <= 2e-2
    st.close()


@pytest.mark.parametrize("recompute", ["none", "selective", "full"])
@pytest.mark.parametrize("sp", [True, False])
def test_stack_memory_equals_total_first_stage(spl, recompute, sp):
    a, h, s, b = TINY["heads"], TINY["hidden"], TINY["seq"], TINY["batch"]
    t = 2
    mem = {}
    for L in (1, 3):
        st = spl.SeqparStack(spl.BlockConfig(**TINY, dropout_p=0.1), t, L, recompute, sp, "bf16")
        mem[L] = st.memory(0)
        ledgers = [st.layers[l].saved_bytes(0)[0] for l in range(L)]
        st.close()
        assert mem[L]["ledger"] == sum(ledgers)
        total = spl.total_first_stage_bytes(a, h, s, b, t, recompute, sp, L)
        if recompute == "full":
            # the reference counts A·sbh per layer regardless of t/SP; the device keeps its shard
            rows = s // t if sp else s
            assert total == L * 2 * s * b * h
            assert mem[L]["ledger"] == L * 2 * rows * b * h
        else:
            assert mem[L]["ledger"] == total
        assert mem[L]["physical_saved"] == mem[L]["ledger"]  # bf16 acts, u8 masks: widths {2, 1}
        assert mem[L]["layer_workspace"] == 0
    assert mem[3]["workspace"] == mem[1]["workspace"]  # one workspace for the whole stack
    assert mem[3]["params"] == 3 * mem[1]["params"]


def test_stack_graph_replay_bit_identical(spl, orc):
    """Replayed CUDA graphs of every layer reproduce the eager stack bit-for-bit."""
    import torch
    L, t = 3, 2
    x, dy, ps = _stack_case(orc, L)
    outs = []
    for graphs in (False, True):
        st = spl.SeqparStack(spl.BlockConfig(**TINY, dropout_p=0.1, seed=42), t, L, "selective", True, "bf16")
        for l in range(L):
            st.layers[l].load_params(ps[l])
            st.layers[l].set_graphs(graphs)
        xs = [torch.from_numpy(u.copy()).to("cuda", torch.bfloat16) for u in np.split(x, t, axis=0)]
        ds = [torch.from_numpy(u.copy()).to("cuda", torch.bfloat16) for u in np.split(dy, t, axis=0)]
        for _ in range(3):
            y = st.forward(xs)
            dx = st.backward(ds)
        outs.append((torch.cat(y).float().cpu(), torch.cat(dx).float().cpu(), st.layers[0].grads()))
        st.close()
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[0][2], outs[1][2])
