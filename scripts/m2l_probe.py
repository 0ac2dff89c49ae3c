"""M2L arithmetic comparison on one FMM plan: fp64 DGEMM vs tcgen05 int8
Ozaki slices (auto from eps, and explicit counts).  N points uniform on the
unit sphere, sources == targets, nd charges N(0,1), pot+grad.  Reports apply
time, M2L stage time, error vs direct on 400 sampled targets and vs the fp64
FMM on all targets.
Usage: python scripts/m2l_probe.py N eps [N eps ...]   (env NDENS=1)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_10743_b200 as b  # noqa: E402
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

nd = int(os.environ.get("NDENS", "1"))
args = sys.argv[1:] or ["1000000", "1e-6"]
for n, eps in zip(args[::2], args[1::2]):
    n, eps = int(float(n)), float(eps)
    rng = np.random.default_rng(105)
    x = rng.standard_normal((n, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    q = rng.standard_normal((nd, n))
    plan = FmmPlan(x, x, eps, m2l="fp64")
    qd = torch.from_numpy(q).cuda()
    idx = rng.choice(n, 400, replace=False)
    ref = b.evaluate_direct(b.FmmSources(x, q), x[idx], ("pot", "grad"))
    base = None
    modes = ["fp64", b.fmm_plan.m2l_slices_for(eps, plan.nrep), "lowrank"] + ([] if os.environ.get("QUICK") else
                                           [s for s in (5, 6, 7, 8)
                                            if s != b.fmm_plan.m2l_slices_for(eps, plan.nrep)])
    for mode in modes:
        plan.set_m2l(mode)
        pot = torch.empty((nd, n), dtype=torch.float64, device="cuda")
        grad = torch.empty((nd, n, 3), dtype=torch.float64, device="cuda")
        plan.apply_device(qd, None, nd, (1 << nd) - 1, 0, 1, pot, grad)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.apply_device(qd, None, nd, (1 << nd) - 1, 0, 1, pot, grad)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        plan.set_timing(True)
        plan.apply_device(qd, None, nd, (1 << nd) - 1, 0, 1, pot, grad)
        plan.set_timing(False)
        st = plan.stage_times()
        p, g = pot.cpu().numpy(), grad.cpu().numpy()
        err = max(np.abs(p[:, idx] - ref.pot).max() / np.abs(ref.pot).max(),
                  np.abs(g[:, idx] - ref.grad).max() / np.abs(ref.grad).max())
        if base is None:
            base = (p, g)
            dev = 0.0
        else:
            dev = max(np.abs(p - base[0]).max() / np.abs(base[0]).max(),
                      np.abs(g - base[1]).max() / np.abs(base[1]).max())
        print(json.dumps({"N": n, "eps": eps, "nd": nd, "rep": plan.rep, "nrep": plan.nrep,
                          "m2l": mode, "slices": plan.m2l_slices, "apply_ms": min(ts),
                          "m2l_ms": st["m2l"], "err_vs_direct_400": err,
                          "dev_vs_fp64_fmm": dev,
                          "ranks": None if mode != "lowrank" else
                          [int(plan.m2l_ranks.max()), float(plan.m2l_ranks.mean())]}), flush=True)
