"""Dev tool (GPU box, run under ncu): selective-layer forwards of the 22B width at equal token
counts and different sequence lengths, to separate per-CTA fixed costs of the attention forward
from its per-key-step cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_05198_b200 as spl  # noqa: E402

for s, b in ((1024, 8), (2048, 4), (4096, 2), (8192, 1)):
    cfg = spl.BlockConfig(64, 6144, s, b, dropout_p=0.1, causal=False, seed=42)
    L = spl.SeqparLayer(cfg, 1, "selective", True, "bf16", check_finite=False)
    L.init_params(1234)
    x = [(torch.rand(L.shard_shape(), device="cuda") * 2 - 1).to(torch.bfloat16)]
    for _ in range(2):
        L.forward(x)
    torch.cuda.synchronize()
    L.close()
    print(s, b, flush=True)
