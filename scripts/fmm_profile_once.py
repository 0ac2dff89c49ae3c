"""One FMM apply (after a warm-up apply) inside NVTX range "fmm" for ncu.
Usage: python scripts/fmm_profile_once.py N eps"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

n, eps = int(float(sys.argv[1])), float(sys.argv[2])
rng = np.random.default_rng(105)
x = rng.standard_normal((n, 3))
x /= np.linalg.norm(x, axis=1, keepdims=True)
plan = FmmPlan(x, x, eps)
q = torch.from_numpy(rng.standard_normal((1, n))).cuda()
pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("fmm")
plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok")
