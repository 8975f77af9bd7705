"""Loader for tests/golden/layer_*.npz — outputs of the reference's OWN block.cpp.

The fixtures are written by oracle/gen_layer_golden.py from oracle/_ref/libref_seqpar.so (the
reference's tensor/block/collectives/rng.cpp compiled unmodified). Inputs are regenerated here
with the RNG pinned by tests/golden/rng_kat.json, exactly as the generator made them
(verify.cpp:115-119 with seed 42, key 0).
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SHAPES = ("toy", "bench_seqpar", "tiny")
WEIGHTS = ("wq", "wk", "wv", "wo", "w1", "w2")
SEED = 42

_CACHE: dict = {}


@dataclass
class GoldenCase:
    shape: str
    name: str
    heads: int
    hidden: int
    seq: int
    batch: int
    t: int
    dropout_p: float
    causal: bool
    key: int
    arrays: dict

    def get(self, k):
        return self.arrays.get(f"{self.name}/{k}")

    def cfg(self, orc):
        return orc.BlockConfig(heads=self.heads, hidden=self.hidden, seq=self.seq,
                               batch=self.batch, dropout_p=self.dropout_p, causal=self.causal,
                               seed=SEED)

    def inputs(self, orc):
        s, b, h = self.seq, self.batch, self.hidden
        x = orc.random_uniform(orc.hash_counter(SEED, 1000 + self.key), (s, b, h), -1.0, 1.0)
        dy = orc.random_uniform(orc.hash_counter(SEED, 2000 + self.key), (s, b, h), -1.0, 1.0)
        p = orc.params_random(h, orc.hash_counter(SEED, 3000 + self.key))
        sums = self.get("input_sums")
        assert np.array_equal(np.array([x.sum(), dy.sum(), p.sum()]), sums), \
            "input generation drifted from the reference RNG"
        return x, dy, p

    def grads(self):
        pre = f"{self.name}/grad/"
        return {k[len(pre):]: v for k, v in self.arrays.items() if k.startswith(pre)}


def load(shape: str) -> dict:
    if shape not in _CACHE:
        with np.load(os.path.join(GOLDEN, f"layer_{shape}.npz")) as z:
            _CACHE[shape] = {k: z[k] for k in z.files}
    return _CACHE[shape]


def cases(shape: str) -> list[GoldenCase]:
    arrs = load(shape)
    a, h, s, b = (int(v) for v in arrs["shape"])
    out = []
    for k in arrs:
        if k.endswith("/meta"):
            name = k[:-len("/meta")]
            t, causal, key = (int(v) for v in arrs[k])
            p = float(arrs[f"{name}/dropout_p"])
            out.append(GoldenCase(shape, name, a, h, s, b, t, p, bool(causal), key,
                                  {kk: v for kk, v in arrs.items() if kk.startswith(name + "/")}))
    return sorted(out, key=lambda c: c.name)


def all_cases():
    return [c for s in SHAPES for c in cases(s)]
