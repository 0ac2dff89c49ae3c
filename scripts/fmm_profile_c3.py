"""BASELINE config 3's FMM (torus 64 x 32, order 7: 458,752 sources ->
114,688 targets, eps 5e-8, ncrit 300) for ncu: plan, one warm-up apply, one
charge pot+grad apply.  python scripts/fmm_profile_c3.py [eps] [ncrit] [xw]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10743_b200 import shapes  # noqa: E402
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 5e-8
ncrit = int(sys.argv[2]) if len(sys.argv) > 2 else 300
geom = shapes.build_torus(7, 64, 32, 2.0, 1.0)
xw = sys.argv[3] if len(sys.argv) > 3 else "lists"
plan = FmmPlan(geom.over_nodes, geom.nodes, eps, ncrit=ncrit, xw=xw)
n, ns = geom.nnodes, geom.noversampled
q = torch.from_numpy(np.random.default_rng(3).standard_normal((1, ns))).cuda()
pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
for _ in range(2):
    plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
torch.cuda.synchronize()
plan.set_timing(True)
plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
torch.cuda.synchronize()
print(plan.stage_times(), plan.work_counts(), flush=True)
