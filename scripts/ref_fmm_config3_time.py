"""Time the reference's own far field at BASELINE config 3 in THIS container
(the reference cannot travel to the GPU box): the two `FmmPlan.apply` calls of
`apply_a3` (operators.py:229-266 -> fmm.py:784-990) on the config-3 torus
(N = 114,688 targets, 458,752 oversampled sources, eps 5e-8), with the plan
build timed apart. Writes profiles/round2/reference_fmm_config3_cpu.json; the
figure is context for bench.py's reference arm, which times exact sums.

  python scripts/ref_fmm_config3_time.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
import lapbel.fmm as fmm  # noqa: E402
from lapbel import shapes  # noqa: E402

t0 = time.time()
disc = shapes.build_torus(7, 64, 32, 2.0, 1.0)
t_geom = time.time() - t0
n, nover = disc.nnodes, disc.noversampled
rng = np.random.default_rng(2)
w = disc.over_weights * rng.standard_normal(nover)
t0 = time.time()
plan = fmm.FmmPlan(disc.over_nodes, disc.nodes, 5e-8)
t_plan = time.time() - t0
print("plan", t_plan, flush=True)
t0 = time.time()
plan.apply(w[None], None, ("pot", "grad"))
t_call1 = time.time() - t0
print("call1", t_call1, flush=True)
ch = np.stack([w, w, np.zeros_like(w)])
dp = np.zeros((3, nover, 3))
dp[2] = w[:, None] * disc.over_normals
t0 = time.time()
plan.apply(ch, dp, ("pot", "grad", "hess"), np.array([True, True, False]),
           np.array([False, False, True]))
t_call2 = time.time() - t0
print("call2", t_call2, flush=True)
out = {"what": "reference lapbel FmmPlan at config 3 (torus 64x32 order 7), eps 5e-8, this "
               "container's CPU (not the GPU box)",
       "N": n, "N_over": nover, "cores": os.cpu_count(), "geometry_s": t_geom,
       "plan_s": t_plan, "fmm_call1_s": t_call1, "fmm_call2_s": t_call2,
       "far_per_apply_s": t_call1 + t_call2}
os.makedirs(os.path.join(ROOT, "profiles", "round2"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "round2", "reference_fmm_config3_cpu.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
