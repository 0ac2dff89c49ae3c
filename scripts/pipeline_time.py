"""Time to solution at BASELINE config 2 through the public API, from a mesh
file: write_mesh -> read_mesh (device geometry) -> LayerOperatorSet (device
near map + corrections) -> solve_laplace_beltrami (A3, GMRES 1e-10).  Each
stage is wall-clock with a device synchronize on both sides; the reference's
own t_q, apply and solve times for the same case are stored in
tests/golden/config2_geom.npz (measured by scripts/make_golden.py in the
survey container).  One warm-up pass first (CUDA context, tables)."""
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_10743_b200 import (LayerOperatorSet, SolveConfig, read_mesh,  # noqa: E402
                                   solve_laplace_beltrami, write_mesh)
from paper_2111_10743_b200.operators import Geometry  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "config2_geom.npz"))
path = os.path.join(tempfile.mkdtemp(), "config2.lbmesh")
write_mesh(path, Geometry.from_arrays(g))


def run():
    t = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    disc = read_mesh(path)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    op = LayerOperatorSet(disc, "a3", float(g["eps"]))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rep = solve_laplace_beltrami(op, g["f"], SolveConfig(
        formulation="a3", eps=float(g["eps"]), eps_gmres=1e-10))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    t["read_mesh_s"] = t1 - t0
    t["operator_setup_s"] = t2 - t1
    t["t_q_s"] = op.t_q
    t["solve_s"] = t3 - t2
    t["n_iter"] = rep.n_iter
    t["total_s"] = t3 - t0
    w = g["weights"]
    d = rep.u.values - g["a3_u"]
    t["u_rel_wl2_vs_reference"] = float(np.sqrt(np.dot(w, d * d) / np.dot(w, g["a3_u"] ** 2)))
    return t


run()
res = run()
res["reference"] = {"t_q_s": float(g["t_q"]), "solve_s": float(g["a3_t_s"]),
                    "apply_s": float(g["a3_t_apply"]), "n_iter": int(len(g["a3_hist"]))}
print(json.dumps(res))
