"""Oracle layer numerics pinned by the reference's own relational suites:
test_seqpar.cpp:120-271 and verify.cpp:74-321 (forward/backward equivalence across t, causal,
finite differences, ledger, recompute bit-equality, comm volume)."""
import numpy as np
import pytest


def toy(orc, **kw):
    cfg = orc.BlockConfig(heads=2, hidden=8, seq=4, batch=1, seed=7)  # test_seqpar.cpp:31-39
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


def rand(orc, key, cfg):
    return orc.random_uniform(key, (cfg.seq, cfg.batch, cfg.hidden), -1.0, 1.0)


def test_ledger_toy(orc):  # test_seqpar.cpp:120-137
    cfg = toy(orc)
    p = orc.params_random(cfg.hidden, 11)
    r = orc.reference_layer(cfg, p, rand(orc, 3, cfg))
    L = r["ledger"]
    tot = lambda names: sum(L[n][1] for n in names)
    assert tot(L) == 1248
    assert tot(["qkv_input", "query", "key", "value", "softmax_out", "softmax_dropout_mask",
                "softmax_dropout_out", "attn_proj_input", "attn_dropout_mask"]) == 512
    assert tot(["mlp_fc1_input", "gelu_input", "mlp_fc2_input", "mlp_dropout_mask"]) == 608
    assert tot(["ln1_input", "ln2_input"]) == 128


def test_zero_in_zero_out(orc):  # test_seqpar.cpp:139-145
    cfg = toy(orc)
    r = orc.reference_layer(cfg, orc.params_zeros(8), np.zeros((4, 1, 8)))
    assert np.all(r["y"] == 0.0)


def test_seqpar_t1_bit_identical(orc):  # test_seqpar.cpp:161-168
    cfg = toy(orc)
    p = orc.params_random(8, 21)
    x = rand(orc, 22, cfg)
    ref = orc.reference_layer(cfg, p, x)
    sp = orc.seqpar_layer(cfg, 1, p, x)
    assert np.array_equal(sp.y, ref["y"])


def test_seqpar_t2_and_ledger(orc):  # test_seqpar.cpp:170-183
    cfg = toy(orc)
    p = orc.params_random(8, 31)
    x = rand(orc, 32, cfg)
    ref = orc.reference_layer(cfg, p, x)
    sp = orc.seqpar_layer(cfg, 2, p, x)
    assert np.max(np.abs(sp.y - ref["y"])) <= 1e-10
    for led in sp.ledgers:
        assert sum(v[1] for v in led.values()) * 2 == sum(v[1] for v in ref["ledger"].values())


def test_causal(orc):  # test_seqpar.cpp:185-199
    cfg = toy(orc, causal=True)
    p = orc.params_random(8, 41)
    x = rand(orc, 42, cfg)
    ref = orc.reference_layer(cfg, p, x, want_interior=True)
    sm = ref["interior"][0, 0, 0]
    for i1 in range(4):
        for i2 in range(i1 + 1, 4):
            assert sm[i1, i2] == 0.0
    sp = orc.seqpar_layer(cfg, 2, p, x)
    assert np.max(np.abs(sp.y - ref["y"])) <= 1e-10


def test_backward_and_w1_locality(orc):  # test_seqpar.cpp:201-232
    cfg = toy(orc, heads=4)
    p = orc.params_random(8, 51)
    x = rand(orc, 52, cfg)
    dy = rand(orc, 53, cfg)
    ref = orc.reference_layer(cfg, p, x, dy)
    sp = orc.seqpar_layer(cfg, 2, p, x, dy)
    assert np.max(np.abs(sp.dx - ref["dx"])) <= 1e-10
    assert np.max(np.abs(sp.grads - ref["grads"])) <= 1e-10
    w1g = orc.unpack(8, ref["grads"])["w1"]
    for r in range(2):
        assert np.max(np.abs(sp.w1_grad_shards[r] - w1g[:, r * 16:(r + 1) * 16])) <= 1e-10


def test_identity_like_block(orc):  # test_seqpar.cpp:234-246
    cfg = toy(orc)
    dy = rand(orc, 61, cfg)
    r = orc.reference_layer(cfg, orc.params_zeros(8), np.zeros((4, 1, 8)), dy)
    assert np.array_equal(r["dx"], dy)
    g = orc.unpack(8, r["grads"])
    assert np.array_equal(g["b2"], dy.reshape(-1, 8).sum(0))
    assert np.array_equal(g["bo"], dy.reshape(-1, 8).sum(0))


def test_recompute_bit_exact(orc):  # test_seqpar.cpp:248-271
    cfg = toy(orc, dropout_p=0.1)
    p = orc.params_random(8, 71)
    x = rand(orc, 72, cfg)
    ref = orc.reference_layer(cfg, p, x, want_interior=True)
    redone = orc.attention_interior(cfg, ref["q"], ref["k"], 0, cfg.heads)
    assert np.array_equal(redone, ref["interior"])
    discarded = 2 * redone[0].size + 2 * redone[2].size + redone[1].size
    assert discarded == 5 * cfg.heads * cfg.seq ** 2 * cfg.batch == 160
    other = toy(orc, dropout_p=0.1, seed=8)
    wrong = orc.attention_interior(other, ref["q"], ref["k"], 0, cfg.heads)
    assert not np.array_equal(wrong[1], ref["interior"][1])


def test_errors(orc):  # test_seqpar.cpp:273-298
    cfg = toy(orc)
    p = orc.params_random(8, 81)
    with pytest.raises(ValueError):
        orc.seqpar_layer(cfg, 3, p, rand(orc, 82, cfg))
    x = rand(orc, 82, cfg)
    x[0, 0, 0] = np.inf
    with pytest.raises(ArithmeticError):
        orc.reference_layer(cfg, p, x)


class CaseRng:  # verify.cpp:31-39
    def __init__(self, orc, key):
        self.orc, self.key, self.counter = orc, key, 0

    def next(self):
        v = self.orc.uniform01(self.key, self.counter)
        self.counter += 1
        return v

    def pick(self, options):
        idx = int(self.next() * len(options))
        return options[min(idx, len(options) - 1)]


def random_toy_config(orc, rng, seed, layer):  # verify.cpp:41-50
    heads = rng.pick([4, 8])
    hidden = heads * rng.pick([2, 3, 4])
    seq = rng.pick([4, 8, 12])
    batch = rng.pick([1, 2, 3])
    return orc.BlockConfig(heads=heads, hidden=hidden, seq=seq, batch=batch, seed=seed, layer_index=layer)


def test_equivalence_suite(orc):  # verify.cpp:107-147 (seed 42, 20 shapes, t in {1,2,4})
    seed = 42
    rng = CaseRng(orc, orc.hash_counter(seed, 2))
    cases = 0
    for shape_idx in range(20):
        cfg = random_toy_config(orc, rng, seed, shape_idx)
        shp = (cfg.seq, cfg.batch, cfg.hidden)
        x = orc.random_uniform(orc.hash_counter(seed, 1000 + shape_idx), shp, -1, 1)
        lw = orc.random_uniform(orc.hash_counter(seed, 2000 + shape_idx), shp, -1, 1)
        p = orc.params_random(cfg.hidden, orc.hash_counter(seed, 3000 + shape_idx))
        ref = orc.reference_layer(cfg, p, x, lw)
        for t in (1, 2, 4):
            if cfg.heads % t or cfg.seq % t:
                continue
            sp = orc.seqpar_layer(cfg, t, p, x, lw)
            if t == 1:
                assert np.array_equal(sp.y, ref["y"])
            assert np.max(np.abs(sp.y - ref["y"])) <= 1e-10
            assert np.max(np.abs(sp.dx - ref["dx"])) <= 1e-10
            assert np.max(np.abs(sp.grads - ref["grads"])) <= 1e-10
            cases += 1
    assert cases > 20


@pytest.mark.parametrize("variant", [0, 1])
def test_finite_difference(orc, variant):  # verify.cpp:159-214
    seed = 42
    cfg = orc.BlockConfig(heads=4, hidden=8, seq=4, batch=1, seed=seed + variant,
                          dropout_p=0.0 if variant == 0 else 0.1, causal=variant == 1)
    t = 2
    shp = (4, 1, 8)
    x = orc.random_uniform(orc.hash_counter(seed, 4000 + variant), shp, -1, 1)
    lw = orc.random_uniform(orc.hash_counter(seed, 5000 + variant), shp, -1, 1)
    p = orc.params_random(8, orc.hash_counter(seed, 6000 + variant))
    res = orc.seqpar_layer(cfg, t, p, x, lw)
    loss = lambda xx, pp: float(np.sum(lw * orc.seqpar_layer(cfg, t, pp, xx).y))
    step, tol = 1e-5, 1e-6
    worst = 0.0
    for i in range(p.size):
        pu, pd_ = p.copy(), p.copy()
        pu[i] += step
        pd_[i] -= step
        fd = (loss(x, pu) - loss(x, pd_)) / (2 * step)
        an = res.grads[i]
        worst = max(worst, abs(fd - an) / max(1.0, abs(fd), abs(an)))
    for i in range(x.size):
        xu, xd = x.copy().reshape(-1), x.copy().reshape(-1)
        xu[i] += step
        xd[i] -= step
        fd = (loss(xu.reshape(shp), p) - loss(xd.reshape(shp), p)) / (2 * step)
        an = res.dx.reshape(-1)[i]
        worst = max(worst, abs(fd - an) / max(1.0, abs(fd), abs(an)))
    assert worst <= tol


def test_byte_ledger_suite(orc):  # verify.cpp:216-251
    seed = 42
    rng = CaseRng(orc, orc.hash_counter(seed, 7))
    for c in range(100):
        cfg = random_toy_config(orc, rng, seed, c)
        shp = (cfg.seq, cfg.batch, cfg.hidden)
        x = orc.random_uniform(orc.hash_counter(seed, 8000 + c), shp, -1, 1)
        p = orc.params_random(cfg.hidden, orc.hash_counter(seed, 9000 + c))
        ref = orc.reference_layer(cfg, p, x)
        total = sum(v[1] for v in ref["ledger"].values())
        bd = orc.layer_component_breakdown(cfg.heads, cfg.hidden, cfg.seq, cfg.batch)["total"]
        eq1 = orc.per_layer_bytes(cfg.heads, cfg.hidden, cfg.seq, cfg.batch, 1, "none", False)
        assert total == bd == eq1
        t = 4 if cfg.seq % 4 == 0 else 2
        if cfg.heads % t:
            continue
        sp = orc.seqpar_layer(cfg, t, p, x)
        eq3 = orc.per_layer_bytes(cfg.heads, cfg.hidden, cfg.seq, cfg.batch, t, "none", True)
        for led in sp.ledgers:
            lt = sum(v[1] for v in led.values())
            assert lt == eq3 and lt * t == eq1


def test_comm_volume_suite(orc):  # verify.cpp:285-321
    seed = 42
    for t in (2, 4):
        cfg = orc.BlockConfig(heads=4, hidden=8, seq=8, batch=2, seed=seed)
        shp = (8, 2, 8)
        x = orc.random_uniform(orc.hash_counter(seed, 12000 + t), shp, -1, 1)
        dy = orc.random_uniform(orc.hash_counter(seed, 13000 + t), shp, -1, 1)
        p = orc.params_random(8, orc.hash_counter(seed, 14000))
        r = orc.seqpar_layer(cfg, t, p, x, dy)
        f, b = r.fwd_comm, r.bwd_comm
        assert f.schedule.all_gathers + b.schedule.all_gathers == 4
        assert f.schedule.reduce_scatters + b.schedule.reduce_scatters == 4
        assert f.schedule.all_reduces == 0 and b.schedule.all_reduces == 0
        assert b.regather.all_gathers == 2 and b.grad_sync.all_reduces == 6
        measured = (f.schedule.ring_elements + b.schedule.ring_elements) * 2
        assert measured == orc.layer_comm_bytes_sp(8, 2, 8, t) == orc.layer_comm_bytes_tp(8, 2, 8, t)
