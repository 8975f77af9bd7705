"""Dev tool (GPU box, under ncu): 22B t=1 no-recompute layer steps (the stored-interior path)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2205_05198_b200 as spl  # noqa: E402
cfg = spl.BlockConfig(64, 6144, 2048, 4, dropout_p=0.1, causal=False, seed=42)
L = spl.SeqparLayer(cfg, 1, "none", True, "bf16", check_finite=False)
L.init_params(1234)
x = [(torch.rand(L.shard_shape(), device="cuda") * 2 - 1).to(torch.bfloat16)]
dy = [(torch.rand(L.shard_shape(), device="cuda") * 2 - 1).to(torch.bfloat16)]
for _ in range(int(os.environ.get("STEPS", "2"))):
    L.forward(x)
    L.backward(dy)
torch.cuda.synchronize()
