"""FMM on the config-3 geometry (sources = oversampled nodes, targets =
nodes): apply time and stage split vs ncrit and eps."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

g = np.load(os.path.join(ROOT, "data", "config3_geom.npz"))
src, tgt = g["over_nodes"], g["nodes"]
ns, nt = src.shape[0], tgt.shape[0]
rng = np.random.default_rng(0)
for eps in (5e-8, 1e-9):
    for ncrit in (120, 300, 600, 1200):
        plan = FmmPlan(src, tgt, eps, ncrit=ncrit)
        for nd, level in ((1, 1), (3, 2)):
            q = torch.from_numpy(rng.standard_normal((nd, ns))).cuda()
            pot = torch.empty((nd, nt), dtype=torch.float64, device="cuda")
            grad = torch.empty((nd, nt, 3), dtype=torch.float64, device="cuda")
            hess = torch.empty((nd, nt, 3, 3), dtype=torch.float64, device="cuda")
            plan.apply_device(q, None, nd, (1 << nd) - 1, 0, level, pot, grad, hess)
            torch.cuda.synchronize()
            plan.set_timing(True)
            plan.apply_device(q, None, nd, (1 << nd) - 1, 0, level, pot, grad, hess)
            st = plan.stage_times()
            plan.set_timing(False)
            print(json.dumps({"eps": eps, "ncrit": ncrit, "nd": nd, "level": level,
                              "total_ms": st["total"],
                              "stages": {k: round(v, 2) for k, v in st.items()},
                              "nbox": int(plan.tree.sizes[0]), "V": int(plan.tree.sizes[6]),
                              "U": int(plan.tree.sizes[7]), "W": int(plan.tree.sizes[8])}),
                  flush=True)
        del plan
