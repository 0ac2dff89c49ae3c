"""GMRES operator-apply time vs N (the second half of the BASELINE metric).

  config 2: icosphere order 7, N = 8,960 (reference-built corrections);
  config 3: torus build_torus(7, 64, 32, 2, 1), N = 114,688: corrections
            built on the device (quadrature.build_correction_set, eps 5e-8;
            the reference's own build takes hours at this size), or with
            --synthetic SYNTHETIC values on the reference's near-map pattern
            (eta 2, cap 256): apply timing only;
  config 4: wavy torus, N = 1,202,940 (same two options; eps 1e-9).
Far field exact (all-pairs) and through the device FMM.  A3 formulation.
Prints JSON lines with the stage split (far 1, SpMV 1, far 2, SpMV 2 + glue)
and the SpMV passes' achieved HBM bandwidth.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_10743_b200 import CorrectionSet, Geometry, LayerOperatorSet  # noqa: E402

try:  # GB/s, the driver-measured copy bandwidth
    HBM = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except (OSError, KeyError, ValueError):
    HBM = 6552.6


def pattern_from_near(g, dev="cuda"):
    """CSR pattern of compute_corrections (quadrature.py:693-698): row i holds
    nb consecutive columns per near patch, columns sorted."""
    nb = int(g["nb"])
    off = torch.from_numpy(np.asarray(g["near_offsets"], dtype=np.int64)).to(dev)
    pat = torch.from_numpy(np.asarray(g["near_patches"], dtype=np.int64)).to(dev)
    n = off.numel() - 1
    cnt = off[1:] - off[:-1]
    row = torch.repeat_interleave(torch.arange(n, device=dev), cnt)
    key = row * (int(pat.max()) + 1) + pat          # sort patches within each row
    pat = pat[torch.argsort(key)]
    cols = (pat[:, None] * nb + torch.arange(nb, device=dev)[None, :]).reshape(-1)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    indptr[1:] = torch.cumsum(cnt * nb, 0)
    return indptr, cols.to(torch.int32)


def run(name, g, cset, eps, far, reps=5, synthetic=False, ncrit=120, m2l="auto"):
    geom = Geometry.from_arrays(g)
    op = LayerOperatorSet(geom, "a3", eps, corrections=cset, far=far, fmm_ncrit=ncrit,
                          fmm_m2l=m2l)
    n = geom.nnodes
    tau = torch.from_numpy(np.random.default_rng(2).standard_normal(n)).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    op.apply_device(tau, out)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply_device(tau, out)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    op.dev.set_timing(True)
    op.apply_device(tau, out)
    st = op.dev.stage_times()
    nnz = int(cset.indices.shape[0])
    fused = op.dev.keep.get("phi_eta") is not None  # pass 2 reads 2 kinds, else 3
    b1 = nnz * (2 * 8 + 4) + 8 * (n + 1)
    b2 = nnz * ((2 if fused else 3) * 8 + 4) + 8 * (n + 1)
    slices = op._plan.m2l_slices if op.far == "fmm" else None
    print(json.dumps({"case": name, "far": op.far, "fused_a3": fused, "eps": eps,
                      "fmm_ncrit": ncrit,
                      "m2l_slices": slices, "N": n,
                      "N_over": geom.noversampled, "nnz_per_kind": nnz,
                      "synthetic_corrections": synthetic, "build": BUILD.get(name),
                      "apply_ms": best,
                      "stages_ms": {"far1": st[0], "spmv1": st[1], "far2": st[2],
                                    "spmv2+glue": st[3], "eta": st[4]},
                      "spmv1_GBps": b1 / (st[1] * 1e-3) / 1e9,
                      "spmv2_GBps": b2 / (st[3] * 1e-3) / 1e9,
                      "spmv1_frac_hbm": b1 / (st[1] * 1e-3) / 1e9 / HBM,
                      "spmv2_frac_hbm": b2 / (st[3] * 1e-3) / 1e9 / HBM}), flush=True)
    del op
    torch.cuda.empty_cache()


BUILD = {}


def corrections(name, g, eps, synthetic, seed):
    if synthetic:
        indptr, idx = pattern_from_near(g)
        gen = torch.Generator(device="cuda").manual_seed(seed)
        vals = {k: 1e-4 * torch.randn(idx.numel(), dtype=torch.float64, device="cuda",
                                      generator=gen)
                for k in ("s", "sprime", "spp_plus_dprime")}
        return CorrectionSet(indptr, idx, vals)
    import time
    from paper_2111_10743_b200 import FORMULATIONS
    from paper_2111_10743_b200.quadrature import LAST_BUILD, build_correction_set, build_near_map
    geom = Geometry.from_arrays(g)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    near = build_near_map(geom, 2.0, cap=256)
    torch.cuda.synchronize()
    t_near = time.perf_counter() - t0
    same = bool(np.array_equal(near.offsets, g["near_offsets"])
                and np.array_equal(near.patches, g["near_patches"]))
    cset, t_q = build_correction_set(geom, near, list(FORMULATIONS["a3"]), eps)
    BUILD[name] = {"eps": eps, "t_near_s": t_near, "near_equal_reference": same,
                   "t_q_s": t_q, "split": dict(LAST_BUILD)}
    print(json.dumps({"case": name, "build": BUILD[name]}), flush=True)
    return cset


if __name__ == "__main__":
    args = sys.argv[1:]
    synthetic = "--synthetic" in args
    only = [a for a in args if not a.startswith("--")]
    c2 = os.path.join(ROOT, "data", "config2.npz")
    if os.path.exists(c2) and (not only or "config2" in only):
        g = dict(np.load(c2))
        cset = CorrectionSet.from_arrays(g)
        run("config2", g, cset, 1e-10, "direct")
        run("config2", g, cset, 1e-10, "fmm")
    c3 = os.path.join(ROOT, "data", "config3_geom.npz")
    if os.path.exists(c3) and (not only or "config3" in only):
        g = dict(np.load(c3))
        cset = corrections("config3", g, 5e-8, synthetic, 3)
        run("config3", g, cset, 5e-8, "fmm", synthetic=synthetic, ncrit=300)
        run("config3", g, cset, 5e-8, "fmm", synthetic=synthetic, ncrit=120)
        run("config3", g, cset, 1e-9, "fmm", synthetic=synthetic, ncrit=300)
        run("config3", g, cset, 5e-8, "direct", reps=2, synthetic=synthetic)
    c4 = os.path.join(ROOT, "data", "config4_geom.npz")
    if os.path.exists(c4) and (not only or "config4" in only):
        g = dict(np.load(c4))
        cset = corrections("config4", g, 1e-9, synthetic, 4)
        torch.cuda.empty_cache()
        run("config4", g, cset, 1e-9, "fmm", reps=2, synthetic=synthetic, ncrit=300)
        run("config4", g, cset, 1e-9, "fmm", reps=2, synthetic=synthetic, ncrit=300,
            m2l="fp64")
