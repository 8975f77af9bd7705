"""dev tool: per-tensor bf16 errors vs the oracle (SPL_ATTN_UMMA=0/1 to compare paths)."""
import os
import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import oracle as orc
import paper_2205_05198_b200 as spl
from test_gpu_layer import make_case, run, rel_l2
for shape, t, causal in [(dict(heads=8, hidden=1024, seq=192, batch=1), 1, True),
                         (dict(heads=8, hidden=1024, seq=256, batch=1), 1, True),
                         (dict(heads=8, hidden=1024, seq=256, batch=1), 1, False)]:
    cfg, x, dy, p = make_case(orc, shape, causal=causal, key=7)
    ref = orc.seqpar_layer(cfg, t, p, x, dy)
    L, y, dx, g = run(spl, cfg, t, p, x, dy, "selective", dtype="bf16")
    G, R = orc.unpack(cfg.hidden, g), orc.unpack(cfg.hidden, ref.grads)
    errs = {k: round(rel_l2(G[k], R[k]), 4) for k in ("wq", "wk", "wv", "bq", "bv", "wo")}
    print(os.environ.get("SPL_ATTN_UMMA", "1"), shape["seq"], causal, "dx", round(rel_l2(dx, ref.dx), 4), errs)
