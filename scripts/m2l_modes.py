"""M2L variants side by side (LB_M2L_MODE: target-major default, fused per
key, staged): FMM stage times at BASELINE config 3 (torus, eps 5e-8) and
config 5 (10^6 sphere, eps 1e-6 / 1e-9), and each variant's agreement with
the staged one.  python scripts/m2l_modes.py"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    sys.path.insert(0, ROOT)
    from paper_2111_10743_b200 import shapes
    from paper_2111_10743_b200.fmm_plan import FmmPlan
    out = {}
    cases = [("config3", None, 5e-8, 300), ("c5_1e6_e6", 1_000_000, 1e-6, 120),
             ("c5_1e6_e9", 1_000_000, 1e-9, 120)]
    for name, n, eps, ncrit in cases:
        if n is None:
            g = shapes.build_torus(7, 64, 32, 2.0, 1.0)
            s, t = g.over_nodes, g.nodes
        else:
            s = shapes.sphere_cloud(n)
            t = s
        plan = FmmPlan(s, t, eps, ncrit=ncrit)
        q = torch.from_numpy(np.random.default_rng(3).standard_normal((2, len(s)))).cuda()
        pot = torch.empty((2, len(t)), dtype=torch.float64, device="cuda")
        grad = torch.empty((2, len(t), 3), dtype=torch.float64, device="cuda")
        for nd in (1, 2):
            for _ in range(2):
                plan.apply_device(q, None, nd, (1 << nd) - 1, 0, 1, pot, grad)
            plan.set_timing(True)
            plan.apply_device(q, None, nd, (1 << nd) - 1, 0, 1, pot, grad)
            torch.cuda.synchronize()
            plan.set_timing(False)
            out[f"{name}_nd{nd}"] = plan.stage_times()
        np.save(os.path.join("/tmp", f"m2l_{os.environ.get('LB_M2L_MODE', 'target')}_{name}.npy"),
                pot.cpu().numpy())
    print(json.dumps(out))
    sys.exit(0)
res = {}
for mode in ("target", "fused", "staged"):
    env = dict(os.environ, LB_M2L_MODE=mode)
    r = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
    if r.returncode:
        print(mode, "FAILED", r.stderr[-2000:])
        continue
    res[mode] = json.loads(r.stdout.strip().splitlines()[-1])
for mode, d in res.items():
    for case, st in d.items():
        print(mode, case, "m2l %.3f ms  total %.3f ms" % (st["m2l"], st["total"]))
for case in ("config3", "c5_1e6_e6", "c5_1e6_e9"):
    ref = np.load(os.path.join("/tmp", f"m2l_staged_{case}.npy"))
    for mode in ("target", "fused"):
        p = os.path.join("/tmp", f"m2l_{mode}_{case}.npy")
        if os.path.exists(p):
            a = np.load(p)
            print(case, mode, "vs staged", float(np.abs(a - ref).max() / np.abs(ref).max()))
