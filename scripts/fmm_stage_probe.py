"""FMM stage split of the two far calls of an A3 apply on a surface point set
(over_nodes -> nodes): call 1 = nd 1 charge, pot+grad; call 2 = nd 2 (charge +
dipole, charge), pot+grad+hess (the two-density A3 call).
Usage: python scripts/fmm_stage_probe.py config3|config4 eps ncrit"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

name, eps, ncrit = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
g = np.load(os.path.join(ROOT, "data", f"{name}_geom.npz"))
src, tgt, nrm = g["over_nodes"], g["nodes"], g["over_normals"]
plan = FmmPlan(src, tgt, eps, ncrit=ncrit)
plan.set_timing(True)
rng = np.random.default_rng(0)
ns, nt = len(src), len(tgt)
c = torch.from_numpy(rng.standard_normal((2, ns))).cuda()
v = torch.zeros((2, ns, 3), dtype=torch.float64, device="cuda")
v[0] = -c[1][:, None] * torch.from_numpy(nrm).cuda()
pot = torch.empty((2, nt), dtype=torch.float64, device="cuda")
grad = torch.empty((2, nt, 3), dtype=torch.float64, device="cuda")
hess = torch.empty((2, nt, 3, 3), dtype=torch.float64, device="cuda")
out = {"case": name, "eps": eps, "ncrit": ncrit, "m2l_slices": plan.m2l_slices}
for label, nd, cm, dm, lv in (("call1", 1, 1, 0, 1), ("call2", 2, 3, 1, 2)):
    for _ in range(2):
        plan.apply_device(c, v, nd, cm, dm, lv, pot, grad, hess)
    torch.cuda.synchronize()
    out[label] = plan.stage_times()
print(json.dumps(out))
