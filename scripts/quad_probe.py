"""Device near-correction build vs the reference's corrections.
Usage: python scripts/quad_probe.py [quad_sphere_o7|opset_sphere_o3|opset_torus_o3|config2|config3]...
Prints per case: near-map equality, build time, per-kind max |diff| / max |ref|."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_10743_b200 import Geometry  # noqa: E402
from paper_2111_10743_b200.operators import KernelKind  # noqa: E402
from paper_2111_10743_b200.quadrature import build_correction_set, build_near_map  # noqa: E402

KINDS = {"s": KernelKind.SINGLE_LAYER, "d": KernelKind.DOUBLE_LAYER,
         "sprime": KernelKind.SPRIME, "grads1": KernelKind.GRAD_S1,
         "grads2": KernelKind.GRAD_S2, "grads3": KernelKind.GRAD_S3,
         "spp_plus_dprime": KernelKind.SPP_PLUS_DPRIME}


def load(name):
    for d in (os.path.join(ROOT, "tests", "golden"), os.path.join(ROOT, "data")):
        for f in (name + ".npz", name + "_geom.npz"):
            p = os.path.join(d, f)
            if os.path.exists(p):
                return dict(np.load(p))
    raise FileNotFoundError(name)


for name in sys.argv[1:] or ["quad_sphere_o7"]:
    g = load(name)
    geom = Geometry.from_arrays(g)
    cap = 256 if name == "config3" else 128
    t0 = time.perf_counter()
    near = build_near_map(geom, float(g.get("near_eta", 2.0)), cap=cap)
    t_near = time.perf_counter() - t0
    same_near = (np.array_equal(near.offsets, g["near_offsets"])
                 and np.array_equal(near.patches, g["near_patches"]))
    out = {"case": name, "N": geom.nnodes, "near_equal": bool(same_near),
           "near_s": t_near, "pairs": int(near.offsets[-1])}
    if "corr_indptr" in g or name == "config3":
        kinds = [k for k in KINDS if "corr_" + k in g] or ["s", "sprime", "spp_plus_dprime"]
        eps = float(g["eps"]) if "eps" in g else 1e-10
        cset, t_q = build_correction_set(geom, near, [KINDS[k] for k in kinds], eps)
        torch.cuda.synchronize()
        # second build: warm timing
        t0 = time.perf_counter()
        cset, t_q = build_correction_set(geom, near, [KINDS[k] for k in kinds], eps)
        torch.cuda.synchronize()
        from paper_2111_10743_b200.quadrature import LAST_BUILD
        out.update({"eps": eps, "t_q_s": time.perf_counter() - t0, "split": dict(LAST_BUILD),
                    "t_q_ref_s": float(g["t_q"]) if "t_q" in g else None,
                    "nnz": cset.nnz})
        if "corr_indptr" in g:
            ip = cset.indptr.cpu().numpy()
            ix = cset.indices.cpu().numpy()
            out["pattern_equal"] = bool(np.array_equal(ip, g["corr_indptr"])
                                        and np.array_equal(ix, g["corr_indices"]))
            errs = {}
            for k in kinds:
                v = cset.values[KINDS[k]].cpu().numpy()
                ref = g["corr_" + k]
                errs[k] = float(np.abs(v - ref).max() / np.abs(ref).max())
                # per-row relative error (rows of very different scale)
                rowmax = np.maximum.reduceat(np.abs(ref), ip[:-1])
                rows = np.repeat(np.arange(len(ip) - 1), np.diff(ip))
                errs[k + "_row"] = float((np.abs(v - ref) / rowmax[rows]).max())
            out["rel_err"] = errs
    print(json.dumps(out), flush=True)
