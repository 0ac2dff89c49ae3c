"""One FMM plan + two applies on a config-5 cloud (for ncu launch lists):
python scripts/fmm_apply_once.py N eps"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

n, eps = int(float(sys.argv[1])), float(sys.argv[2])
rng = np.random.default_rng(105)
x = rng.standard_normal((n, 3))
x /= np.linalg.norm(x, axis=1)[:, None]
q = torch.from_numpy(rng.standard_normal((1, n))).cuda()
plan = FmmPlan(x, x, eps)
pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
for _ in range(2):
    plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
torch.cuda.synchronize()
plan.set_timing(True)
plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
print(plan.stage_times(), flush=True)
