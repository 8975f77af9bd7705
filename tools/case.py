"""Run one sweep case (dev tool, GPU box): python tools/case.py CONFIG T RECOMPUTE [sp]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import paper_2205_05198_b200 as spl  # noqa: E402
from sweep import run_case  # noqa: E402

torch.cuda.set_device(0)
cfg, t, rc = sys.argv[1], int(sys.argv[2]), sys.argv[3]
sp = len(sys.argv) < 5 or sys.argv[4] != "nosp"
r = run_case(spl, torch, cfg, t, rc, sp, 1, 1)
print(r["per_gpu_compute_ms"], r["class_ms_per_gpu"])
