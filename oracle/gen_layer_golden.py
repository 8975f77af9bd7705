"""Generate tests/golden/layer_*.npz from the reference's OWN seqpar harness.

TEST INFRASTRUCTURE. Run here (in the container that has /root/reference):
    make -C oracle ref && python -m oracle.gen_layer_golden
oracle/_ref/libref_seqpar.so is /root/reference/proj/core/src/seqpar/{tensor,block,collectives,
rng}.cpp compiled unmodified (oracle/Makefile `ref`), so every array written here is an output
of the reference's block.cpp, not of our restatement.

Inputs follow verify.cpp:115-119 (seed 42, case key k): x = random_uniform(hash_counter(seed,
1000+k), {s,b,h}, -1, 1), dy = loss weights random_uniform(hash_counter(seed, 2000+k)), params =
LayerParams::random(cfg, hash_counter(seed, 3000+k)). The inputs are NOT stored — the tests
regenerate them with the RNG that tests/golden/rng_kat.json pins bit-exactly — but their sums
are, so drift in input generation fails loudly instead of as a numerics mismatch.

Shapes: toy (a=2 h=8 s=4 b=1), bench_seqpar (a=8 h=64 s=32 b=2, bench_seqpar.cpp:44), tiny
(a=8 h=256 s=128 b=2, BASELINE configs[0]). Per case: y, dx, the 16 assembled parameter
gradients (block.cpp:730-746), per-rank ledgers (elements, bytes), forward/backward CommLog
counters; for the first two p > 0 cases the attention interior (softmax_out fp64, mask u8, dropout_out fp64).
Storage: fp64 throughout except the tiny shape's 6 weight gradients (fp32, 786k values) and
tiny y/dx beyond the first case (fp32) to keep the fixtures small; fp32 storage is 6e-8
relative, far inside the GPU tolerances (1e-5 / 1e-4 fp32 path).
"""
from __future__ import annotations

import itertools
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

OUT = os.path.join(HERE, "..", "tests", "golden")
SEED = 42
WEIGHTS = ("wq", "wk", "wv", "wo", "w1", "w2")

SHAPES = {
    "toy": dict(heads=2, hidden=8, seq=4, batch=1),
    "bench_seqpar": dict(heads=8, hidden=64, seq=32, batch=2),
    "tiny": dict(heads=8, hidden=256, seq=128, batch=2),
}
CASES = {
    "toy": list(itertools.product((1, 2), (0.0, 0.1), (False, True))),
    "bench_seqpar": [(1, 0.1, False), (2, 0.1, True), (4, 0.1, False), (4, 0.0, True),
                     (1, 0.0, False), (2, 0.1, False)],
    "tiny": [(1, 0.1, False), (2, 0.1, True), (4, 0.0, False)],
}


def case_name(t, p, c):
    return f"t{t}_p{int(round(p * 10))}_c{int(c)}"


def counters(log):
    return np.array([[getattr(log, tag).all_gathers, getattr(log, tag).reduce_scatters,
                      getattr(log, tag).all_reduces, getattr(log, tag).ring_elements]
                     for tag in ("schedule", "regather", "grad_sync")], np.int64)


def generate(shape_name: str) -> dict:
    shape = SHAPES[shape_name]
    out = {}
    key = 0
    for ci, (t, p, causal) in enumerate(CASES[shape_name]):
        if shape["heads"] % t or shape["seq"] % t:
            continue
        cfg = O.BlockConfig(**shape, dropout_p=p, causal=causal, seed=SEED)
        s, b, h = cfg.seq, cfg.batch, cfg.hidden
        x = R.random_uniform(R.hash_counter(SEED, 1000 + key), (s, b, h), -1.0, 1.0)
        dy = R.random_uniform(R.hash_counter(SEED, 2000 + key), (s, b, h), -1.0, 1.0)
        params = R.params_random(h, R.hash_counter(SEED, 3000 + key))
        r = R.seqpar_layer(cfg, t, params, x, dy, want_interior=p > 0)
        n = case_name(t, p, causal)
        big = shape_name == "tiny"
        act = np.float32 if big and ci > 0 else np.float64
        out[f"{n}/y"] = r.y.astype(act)
        out[f"{n}/dx"] = r.dx.astype(act)
        grads = O.unpack(h, r.grads)
        for name, g in grads.items():
            if big and name in WEIGHTS:
                if ci == 0:
                    out[f"{n}/grad/{name}"] = g.astype(np.float32)
            else:
                out[f"{n}/grad/{name}"] = g.copy()
        out[f"{n}/ledger"] = np.array([[r.ledgers[q][e] for e in O.LEDGER_NAMES]
                                       for q in range(t)], np.int64)  # [t, 15, (elems, bytes)]
        out[f"{n}/comm_fwd"] = counters(r.fwd_comm)
        out[f"{n}/comm_bwd"] = counters(r.bwd_comm)
        out[f"{n}/input_sums"] = np.array([x.sum(), dy.sum(), params.sum()])
        if p > 0 and not big and ci < 2:
            out[f"{n}/interior/softmax_out"] = r.interior[0].copy()
            out[f"{n}/interior/mask"] = r.interior[1].astype(np.uint8)
            out[f"{n}/interior/dropout_out"] = r.interior[2].copy()
        elif p > 0 and ci == 0:
            # tiny: the mask bit-exactly (u8) and the softmax at fp32.
            out[f"{n}/interior/mask"] = r.interior[1].astype(np.uint8)
            out[f"{n}/interior/softmax_out"] = r.interior[0].astype(np.float32)
        out[f"{n}/meta"] = np.array([t, int(causal), key], np.int64)
        out[f"{n}/dropout_p"] = np.array(p)
    out["shape"] = np.array([shape["heads"], shape["hidden"], shape["seq"], shape["batch"]], np.int64)
    return out


def main():
    if not R.available():
        raise SystemExit("build oracle/_ref first: make -C oracle ref")
    os.makedirs(OUT, exist_ok=True)
    for name in SHAPES:
        arrs = generate(name)
        path = os.path.join(OUT, f"layer_{name}.npz")
        np.savez_compressed(path, **arrs)
        print(f"{path}: {len(arrs)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
