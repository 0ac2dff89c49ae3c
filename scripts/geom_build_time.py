"""Time the device geometry build (lb_geom_build via build_from_coefficients)
at config-2 size and at ~config-4 patch counts (config-2 charts tiled)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2111_10743_b200 import build_from_coefficients
from paper_2111_10743_b200.surface import geometry_tables

g = np.load("tests/golden/config2_geom.npz")
out = []
for order, reps in ((7, 1), (7, 84)):
    cx, cu, cv = (np.tile(g[k], (reps, 1, 1)) for k in ("coeffs_x", "coeffs_dxdu", "coeffs_dxdv"))
    geometry_tables(order)
    build_from_coefficients(order, cx, cu, cv)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = build_from_coefficients(order, cx, cu, cv)
    t1 = time.perf_counter()
    out.append({"order": order, "npatches": cx.shape[0], "N": d.nnodes,
                "N_over": d.noversampled, "build_s_incl_h2d_d2h": t1 - t0})
for o in out:
    print(json.dumps(o))
