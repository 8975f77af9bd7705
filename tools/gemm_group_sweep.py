"""Raster-group sweep of the pair GEMM at the 22B layer's 12 shapes (dev tool, GPU box): ms per
launch for each forced SPL_GEMM_GROUP next to the picked group, two interleaved passes.

    python tools/gemm_group_sweep.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_bench import bench, layer_cases  # noqa: E402

GROUPS = [0, 2, 3, 4, 6, 8, 12, 16, 24, 32]
res = {}
for p in range(2):
    for name, M, N, K, amn, bmn, epi in layer_cases(6144, 8192, 1):
        for gm in GROUPS:
            os.environ["SPL_GEMM_GROUP"] = str(gm)
            _, ms = bench(M, N, K, amn, bmn, epi, reps=10)
            res.setdefault((name, gm), []).append(ms)
for name, *_ in layer_cases(6144, 8192, 1):
    row = {gm: min(res[(name, gm)]) for gm in GROUPS}
    best = min(row, key=row.get)
    print(f"{name:11s} picked {row[0]*1e3:7.1f} us  best g={best:2d} {row[best]*1e3:7.1f} us  " +
          " ".join(f"{gm}:{row[gm]*1e3:.0f}" for gm in GROUPS[1:]), flush=True)
