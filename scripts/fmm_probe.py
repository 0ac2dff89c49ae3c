"""Config-5 style FMM timing: N points uniform on the unit sphere, sources ==
targets, nd=1 charges N(0,1), pot+grad; plan time, apply time (CUDA events),
stage breakdown, accuracy vs direct on 200 sampled targets.
Usage: python scripts/fmm_probe.py N eps [N eps ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_10743_b200 as b  # noqa: E402
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

args = sys.argv[1:] or ["1000000", "1e-6"]
for n, eps in zip(args[::2], args[1::2]):
    n, eps = int(float(n)), float(eps)
    rng = np.random.default_rng(105)
    x = rng.standard_normal((n, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    q = rng.standard_normal((1, n))
    t0 = time.perf_counter()
    plan = FmmPlan(x, x, eps)
    t_plan = time.perf_counter() - t0
    qd = torch.from_numpy(q).cuda()
    pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
    grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
    plan.apply_device(qd, None, 1, 1, 0, 1, pot, grad)  # first apply uploads the plan
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.apply_device(qd, None, 1, 1, 0, 1, pot, grad)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    plan.set_timing(True)
    plan.apply_device(qd, None, 1, 1, 0, 1, pot, grad)
    stages = plan.stage_times()
    idx = rng.choice(n, 200, replace=False)
    ref = b.evaluate_direct(b.FmmSources(x, q), x[idx], ("pot", "grad"))
    p = pot.cpu().numpy()[:, idx]
    g = grad.cpu().numpy()[:, idx]
    err = max(np.abs(p - ref.pot).max() / np.abs(ref.pot).max(),
              np.abs(g - ref.grad).max() / np.abs(ref.grad).max())
    t = min(ts)
    print(json.dumps({"N": n, "eps": eps, "rep": plan.rep, "m": plan.m, "plan_s": t_plan,
                      "apply_s": t, "effective_pairs_per_s": n * (n - 1) / t,
                      "err_vs_direct_200": err, "stages_ms": stages,
                      "tree": {"nbox": int(plan.tree.sizes[0]), "V": int(plan.tree.sizes[6]),
                               "U": int(plan.tree.sizes[7])}}), flush=True)
