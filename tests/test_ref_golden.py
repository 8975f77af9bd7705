"""The fp64 restatement (oracle/liboracle.so) against the reference ITSELF.

Two sources of truth, both produced by the reference's own block.cpp / tensor.cpp /
collectives.cpp / rng.cpp (compiled unmodified into oracle/_ref/libref_seqpar.so):
  * the committed fixtures tests/golden/layer_*.npz (always available, also on the GPU box);
  * the compiled library itself, when it was built here (`make -C oracle ref`), for the
    randomised verify.cpp-style shapes and the per-function entry points.
Tolerance vs fp64 fixtures: max-abs <= 1e-12 * max|ref| (the two sum in different orders);
fp32-stored fixture arrays: 1e-6 relative. Masks, ledgers and CommLog counters: exact.
"""
import numpy as np
import pytest

import golden_layer as G

CASES = G.all_cases()


def close(got, want, what, floor=1e-300):
    """max-abs error within tol * max|want|; `floor` lifts the scale for tensors whose exact
    value is ~0 (the key-bias gradient: softmax is shift-invariant, so it is rounding noise)."""
    want = np.asarray(want)
    tol = 1e-12 if want.dtype == np.float64 else 2e-6
    scale = max(float(np.max(np.abs(want))), floor)
    err = float(np.max(np.abs(got - want.astype(np.float64))))
    assert err <= tol * scale, (what, err / scale)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c.shape}-{c.name}")
def test_oracle_matches_reference_golden(orc, case):
    cfg = case.cfg(orc)
    x, dy, p = case.inputs(orc)
    r = orc.seqpar_layer(cfg, case.t, p, x, dy, want_interior=case.dropout_p > 0)
    close(r.y, case.get("y"), "y")
    close(r.dx, case.get("dx"), "dx")
    got = orc.unpack(cfg.hidden, r.grads)
    gg = case.grads()
    assert len(gg) in (10, 16)
    floor = max(float(np.max(np.abs(v))) for v in gg.values())
    for name, want in gg.items():
        close(got[name], want, name, floor=1e-3 * floor)
    led = np.array([[r.ledgers[q][e] for e in orc.LEDGER_NAMES] for q in range(case.t)])
    assert np.array_equal(led, case.get("ledger"))
    for log, key in ((r.fwd_comm, "comm_fwd"), (r.bwd_comm, "comm_bwd")):
        got_c = np.array([[getattr(log, tag).all_gathers, getattr(log, tag).reduce_scatters,
                           getattr(log, tag).all_reduces, getattr(log, tag).ring_elements]
                          for tag in ("schedule", "regather", "grad_sync")])
        assert np.array_equal(got_c, case.get(key)), key
    if case.get("interior/mask") is not None:
        assert np.array_equal(r.interior[1].astype(np.uint8), case.get("interior/mask"))
        close(r.interior[0], case.get("interior/softmax_out"), "softmax_out")
    if case.get("interior/dropout_out") is not None:
        close(r.interior[2], case.get("interior/dropout_out"), "dropout_out")


def test_golden_covers_the_matrix():
    names = {(c.shape, c.t, c.dropout_p > 0, c.causal) for c in CASES}
    assert {("toy", t, p, c) for t in (1, 2) for p in (False, True) for c in (False, True)} <= names
    assert {("bench_seqpar", 4, True, False), ("bench_seqpar", 2, True, True)} <= names
    assert {("tiny", 1, True, False), ("tiny", 2, True, True), ("tiny", 4, False, False)} <= names


# ------------------------------------------------------------- direct, against oracle/_ref
@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref/libref_seqpar.so not built (needs /root/reference)")
    return R


def test_verify_style_random_shapes_vs_reference(orc, ref):
    """verify.cpp:107-147's 20 random toy configurations, restatement vs reference."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_layer import CaseRng, random_toy_config
    seed = 42
    rng = CaseRng(orc, orc.hash_counter(seed, 2))
    n = 0
    for idx in range(20):
        cfg = random_toy_config(orc, rng, seed, idx)
        shp = (cfg.seq, cfg.batch, cfg.hidden)
        x = orc.random_uniform(orc.hash_counter(seed, 1000 + idx), shp, -1, 1)
        lw = orc.random_uniform(orc.hash_counter(seed, 2000 + idx), shp, -1, 1)
        p = orc.params_random(cfg.hidden, orc.hash_counter(seed, 3000 + idx))
        assert np.array_equal(p, ref.params_random(cfg.hidden, orc.hash_counter(seed, 3000 + idx)))
        want = ref.reference_layer(cfg, p, x, lw, want_interior=True)
        got = orc.reference_layer(cfg, p, x, lw, want_interior=True)
        for k in ("y", "dx", "grads", "q", "k"):
            close(got[k], want[k], k)  # grads: one packed vector, scale = its max
        assert np.array_equal(got["interior"][1], want["interior"][1])
        assert got["ledger"] == want["ledger"]
        for t in (1, 2, 4):
            if cfg.heads % t or cfg.seq % t:
                continue
            a = orc.seqpar_layer(cfg, t, p, x, lw)
            b = ref.seqpar_layer(cfg, t, p, x, lw)
            close(a.y, b.y, "y")
            close(a.dx, b.dx, "dx")
            close(a.grads, b.grads, "grads")
            close(a.w1_grad_shards, b.w1_grad_shards, "w1 shards")
            assert a.ledgers == b.ledgers
            n += 1
    assert n >= 20


def test_attention_interior_head_slice_vs_reference(orc, ref):
    """attention_interior(q, k, cfg, head_offset, local_heads) (block.cpp:381-417)."""
    cfg = orc.BlockConfig(heads=8, hidden=64, seq=32, batch=2, dropout_p=0.1, causal=True)
    for off, lh in ((0, 8), (2, 2), (6, 2), (4, 4)):
        q = orc.random_uniform(11 + off, (32, 2, lh * 8), -1, 1)
        k = orc.random_uniform(12 + off, (32, 2, lh * 8), -1, 1)
        a = orc.attention_interior(cfg, q, k, off, lh)
        b = ref.attention_interior(cfg, q, k, off, lh)
        assert np.array_equal(a[1], b[1])
        close(a[0], b[0], "softmax")
        close(a[2], b[2], "dropout_out")


def test_collectives_vs_reference(ref):
    """all_gather / reduce_scatter / all_reduce + CommLog ring elements (collectives.cpp:21-73)."""
    rs = np.random.default_rng(0)
    for t in (1, 2, 4):
        shards = rs.standard_normal((t, 4, 3, 8))
        full, log = ref.all_gather(shards, 0)
        assert np.array_equal(full, np.concatenate(list(shards), 0))
        assert log.schedule.all_gathers == 1
        assert log.schedule.ring_elements == (full.size // t) * (t - 1)
        parts, log = ref.reduce_scatter(shards, 1 if t == 1 else 0, tag=1)
        acc = shards[0].copy()
        for r in range(1, t):
            acc = acc + shards[r]
        assert np.array_equal(np.concatenate(list(parts), 1 if t == 1 else 0), acc)
        assert log.regather.reduce_scatters == 1
        tot, log = ref.all_reduce(shards, tag=2)
        assert np.array_equal(tot, acc)
        assert log.grad_sync.ring_elements == 2 * (acc.size // t) * (t - 1)


def test_comm_bytes_vs_reference(orc, ref):
    for (s, b, h, t) in ((2048, 4, 6144, 8), (2048, 1, 12288, 2), (128, 2, 256, 1)):
        assert orc.layer_comm_bytes_tp(s, b, h, t) == ref.layer_comm_bytes_tp(s, b, h, t, 2)
        assert orc.layer_comm_bytes_sp(s, b, h, t) == ref.layer_comm_bytes_sp(s, b, h, t, 2)
