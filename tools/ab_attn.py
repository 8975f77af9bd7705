"""A/B helper (dev tool, GPU box): one 22B-shape selective layer step's dx / grads digest and
the attention-class time under the current environment (kernel-variant switches)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_05198_b200 as spl  # noqa: E402

cfg = spl.BlockConfig(64, 6144, 2048, 4, dropout_p=0.1, causal=False, seed=42)
L = spl.SeqparLayer(cfg, 1, "selective", True, "bf16", check_finite=False)
L.init_params(1234)
g = torch.Generator(device="cuda:0").manual_seed(100)
x = [(torch.rand(L.shard_shape(), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)]
dy = [(torch.rand(L.shard_shape(), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)]
L.forward(x)
dx = L.backward(dy)
torch.cuda.synchronize()
h = hashlib.sha256(dx[0].view(torch.int16).cpu().numpy().tobytes()).hexdigest()[:16]
gh = hashlib.sha256(L.grads().tobytes()).hexdigest()[:16]
L.profile(True)
for _ in range(5):
    L.forward(x)
    L.backward(dy)
p = L.profile_read()
L.profile(False)
env = {k: v for k, v in os.environ.items() if k.startswith("SPL_ATTN")}
print(json.dumps({"env": env, "dx": h, "grads": gh, "attn_ms": p["attention"]["ms"] / 5}))
