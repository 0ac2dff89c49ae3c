"""BASELINE config 5's FMM (10^6 points on the sphere) for ncu: plan, two
warm-up applies, one timed charge pot+grad apply.
python scripts/fmm_profile_c5.py [eps] [n] [xw]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10743_b200 import shapes  # noqa: E402
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-9
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
xw = sys.argv[3] if len(sys.argv) > 3 else "lists"
x = shapes.sphere_cloud(n)
plan = FmmPlan(x, x, eps, xw=xw)
q = torch.from_numpy(np.random.default_rng(5).standard_normal((1, n))).cuda()
pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
for _ in range(2):
    plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
torch.cuda.synchronize()
plan.set_timing(True)
plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
torch.cuda.synchronize()
print(plan.stage_times(), plan.work_counts(), flush=True)
