"""One A3 apply with the FMM far field on config 3 (synthetic correction
values on the reference's near-map pattern), after a warm-up apply, for ncu
captures of the FMM leaf kernels.  Usage: python scripts/leaf_profile_once.py [eps]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import apply_vs_n  # noqa: E402
from paper_2111_10743_b200 import Geometry, LayerOperatorSet  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-9
g = dict(np.load(os.path.join(ROOT, "data", "config3_geom.npz")))
cset = apply_vs_n.corrections("config3", g, eps, True, 3)
op = LayerOperatorSet(Geometry.from_arrays(g), "a3", eps, corrections=cset, far="fmm", fmm_ncrit=300)
tau = torch.from_numpy(np.random.default_rng(2).standard_normal(g["nodes"].shape[0])).cuda()
out = torch.empty_like(tau)
op.apply_device(tau, out)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("apply")
op.apply_device(tau, out)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok")
