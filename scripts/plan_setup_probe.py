"""Setup cost of an FMM evaluation on the device (config 5 clouds): plan
construction (keys/sort/tree/lists + unit operators + M2L factors) and the
first apply (device state build) vs a steady-state apply.  One JSON line per
case; used for profiles/round1/plan_setup.md."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

cases = [(1_000_000, 1e-6), (1_000_000, 1e-9), (10_000_000, 1e-6), (10_000_000, 1e-9)]
if len(sys.argv) > 1:
    cases = [(int(float(a.split(":")[0])), float(a.split(":")[1])) for a in sys.argv[1:]]
for n, eps in cases:
    rng = np.random.default_rng(105)
    x = rng.standard_normal((n, 3))
    x /= np.linalg.norm(x, axis=1)[:, None]
    q = rng.standard_normal((1, n))
    FmmPlan(x[:1000], x[:1000], eps)  # unit operators (lru cache), CUDA context
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = FmmPlan(x, x, eps)
    t_plan = time.perf_counter() - t0
    qd = torch.from_numpy(q).cuda()
    pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
    grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.apply_device(qd, None, 1, 1, 0, 1, pot, grad)
    torch.cuda.synchronize()
    t_first = time.perf_counter() - t0
    t0 = time.perf_counter()
    plan.apply_device(qd, None, 1, 1, 0, 1, pot, grad)
    torch.cuda.synchronize()
    t_second = time.perf_counter() - t0
    print(json.dumps({"case": f"fmm N={n} eps={eps}", "plan_s": t_plan,
                      "first_apply_s": t_first, "apply_s": t_second,
                      "setup_s": t_plan + t_first - t_second,
                      "setup_ms": plan.setup_times()}),
          flush=True)
    del plan
    torch.cuda.empty_cache()
