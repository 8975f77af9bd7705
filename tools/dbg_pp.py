"""Debug helper (GPU box): layer forward y with SPL_ATTN_FWD_PP=0 vs 1 at a small shape; prints
which token rows differ."""
import os, subprocess, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
shape = json.loads(sys.argv[1]) if len(sys.argv) > 1 else dict(heads=8, hidden=768, seq=256, batch=2)
if os.environ.get("DBG_CHILD"):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2205_05198_b200 as spl
    cfg = spl.BlockConfig(shape["heads"], shape["hidden"], shape["seq"], shape["batch"], dropout_p=float(os.environ.get("DBG_P", "0.1")), causal=bool(int(os.environ.get("DBG_CAUSAL", "0"))), seed=42)
    L = spl.SeqparLayer(cfg, 1, "selective", True, "bf16", check_finite=False)
    L.init_params(1234)
    g = torch.Generator(device="cuda:0").manual_seed(100)
    x = [(torch.rand(L.shard_shape(), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)]
    y = L.forward(x)[0].float().cpu().numpy()
    np.save(os.environ["DBG_OUT"], y)
    sys.exit(0)
ys = []
for v in ("0", "1"):
    out = f"/tmp/dbg_y{v}.npy"
    env = dict(os.environ, DBG_CHILD="1", SPL_ATTN_FWD_PP=v, DBG_OUT=out)
    r = subprocess.run([sys.executable, __file__, json.dumps(shape)], env=env, timeout=120)
    print("child", v, r.returncode)
    ys.append(np.load(out))
a, b = ys
print("finite", np.isfinite(a).all(), np.isfinite(b).all())
d = np.abs(a - b).reshape(shape["seq"], shape["batch"], -1).max(-1)
print("max diff", np.nanmax(d), "rel", np.nanmax(d) / np.abs(a).max())
bad = np.argwhere(~(d < 0.05 * np.abs(a).max()))
print("bad rows (s, b):", len(bad), bad[:20].tolist(), bad[-5:].tolist())
