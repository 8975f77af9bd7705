"""A/B helper (dev tool, GPU box): one 22B-shape selective layer step's dx / grads digest and
the attention-class time under the current environment (kernel-variant switches)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_05198_b200 as spl  # noqa: E402

# AB_SHAPE: 22B (default, head_dim 96), 175B (head_dim 128), 530B (head_dim 160, t = 8 heads)
shape = os.environ.get("AB_SHAPE", "22B")
a_, h_, b_, t_ = {"22B": (64, 6144, 4, 1), "175B": (96, 12288, 1, 1), "530B": (128, 20480, 1, 8)}[shape]
cfg = spl.BlockConfig(a_, h_, 2048, b_, dropout_p=0.1, causal=False, seed=42)
L = spl.SeqparLayer(cfg, t_, "selective", True, "bf16", check_finite=False)  # t_ simulated ranks
L.init_params(1234)
g = torch.Generator(device="cuda:0").manual_seed(100)
x = [(torch.rand(L.shard_shape(), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(t_)]
dy = [(torch.rand(L.shard_shape(), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(t_)]
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
