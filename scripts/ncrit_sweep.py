"""FMM leaf capacity sweep at BASELINE config 3 (torus 64 x 32, eps 5e-8):
event-timed nd = 1 (pot + grad) and nd = 2 applies per ncrit.
python scripts/ncrit_sweep.py [ncrit ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10743_b200 import shapes  # noqa: E402
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

g = shapes.build_torus(7, 64, 32, 2.0, 1.0)
s, t = g.over_nodes, g.nodes
q = torch.from_numpy(np.random.default_rng(3).standard_normal((2, len(s)))).cuda()
pot = torch.empty((2, len(t)), dtype=torch.float64, device="cuda")
grad = torch.empty((2, len(t), 3), dtype=torch.float64, device="cuda")
for ncrit in [int(a) for a in sys.argv[1:]] or [150, 200, 300, 400, 500, 700]:
    plan = FmmPlan(s, t, 5e-8, ncrit=ncrit, xw=os.environ.get("LB_XW", "direct"))
    row = {"ncrit": ncrit}
    for nd in (1, 2):
        for _ in range(2):
            plan.apply_device(q, None, nd, (1 << nd) - 1, 0, 1, pot, grad)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            plan.apply_device(q, None, nd, (1 << nd) - 1, 0, 1, pot, grad)
        e1.record()
        torch.cuda.synchronize()
        row[f"nd{nd}_ms"] = e0.elapsed_time(e1) / 3
        plan.set_timing(True)
        plan.apply_device(q, None, nd, (1 << nd) - 1, 0, 1, pot, grad)
        torch.cuda.synchronize()
        plan.set_timing(False)
        row[f"nd{nd}_stages"] = {k: round(v, 3) for k, v in plan.stage_times().items()}
    print(json.dumps(row), flush=True)
    del plan
