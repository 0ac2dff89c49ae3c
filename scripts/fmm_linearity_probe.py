"""Additivity of the operator applies with the FMM far field:
|A(x + y) - A(x) - A(y)| / |A(x)| per path (diagnostic)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from conftest import golden  # noqa: E402
from paper_2111_10743_b200 import KernelKind, LayerOperatorSet  # noqa: E402

g = golden("opset_torus_o3.npz")
rng = np.random.default_rng(0)
n = len(g["tau"])
x, y = rng.standard_normal(n), rng.standard_normal(n)


def add(f):
    ax, ay, axy = f(x), f(y), f(x + y)
    return np.abs(axy - ax - ay).max() / np.abs(ax).max()


for far in ("direct", "fmm"):
    op = LayerOperatorSet.from_bundle(g, "a3", eps=5e-8, far=far, fmm_m2l="fp64")
    print(far, "A3", add(op.apply))
    for k in (KernelKind.SINGLE_LAYER, KernelKind.SPRIME, KernelKind.SPP_PLUS_DPRIME):
        if k in op.corrections:
            print(far, k.value, add(lambda v: op.apply_layer(k, v)))
    if far == "fmm":
        op.dev.set_fmm_a3(False)
        print(far, "A3 three densities", add(op.apply))

from paper_2111_10743_b200 import FmmPlan  # noqa: E402
src, tgt = np.asarray(g["over_nodes"]), np.asarray(g["nodes"])
for ncrit in (120, 30):
    for eps in (5e-8, 1e-9):
        plan = FmmPlan(src, tgt, eps, ncrit=ncrit, m2l="fp64")
        c1, c2 = rng.standard_normal((1, len(src))), rng.standard_normal((1, len(src)))
        r1, r2, r3 = (plan.apply(c, None, ("pot",)).pot for c in (c1, c2, c1 + c2))
        print("raw plan torus", ncrit, eps, np.abs(r3 - r1 - r2).max() / np.abs(r1).max(),
              "levels", getattr(plan, "nlevels", None))
