import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import golden
from paper_2111_10743_b200 import KernelKind, LayerOperatorSet
import torch
g = golden("opset_torus_o3.npz")
rng = np.random.default_rng(0)
n = len(g["tau"])
x, y = rng.standard_normal(n), rng.standard_normal(n)
op = LayerOperatorSet.from_bundle(g, "a3", eps=5e-8, far="fmm", fmm_m2l="fp64")
S = KernelKind.SINGLE_LAYER
a1 = op.apply_layer(S, x)
op.apply_layer(S, y)
a2 = op.apply_layer(S, x)
print("history dependence S", np.abs(a2 - a1).max() / np.abs(a1).max())
torch.cuda.synchronize()
op.apply_layer(S, y); torch.cuda.synchronize()
a3 = op.apply_layer(S, x)
print("with sync", np.abs(a3 - a1).max() / np.abs(a1).max())

from paper_2111_10743_b200 import FmmPlan
oi = np.asarray(g["over_interp"]); nb = oi.shape[1]
def ovs(v):
    return (v.reshape(-1, nb) @ oi.T).ravel() * np.asarray(g["over_weights"])
plan = op._plan
for name, cx, cy in (("oversampled", ovs(x), ovs(y)),
                     ("random", rng.standard_normal(len(g["over_nodes"])), rng.standard_normal(len(g["over_nodes"])))):
    r1, r2, r3 = (plan.apply(c[None], None, ("pot",)).pot for c in (cx, cy, cx + cy))
    print("op plan", name, np.abs(r3 - r1 - r2).max() / np.abs(r1).max())
