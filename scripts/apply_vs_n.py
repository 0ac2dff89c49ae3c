"""GMRES operator-apply time vs N (the second half of the BASELINE metric).

  config 2: icosphere order 7, N = 8,960 (reference-built corrections);
  config 3: torus build_torus(7, 64, 32, 2, 1), N = 114,688, the reference's
            near map (eta 2, cap 256) as the CSR pattern with SYNTHETIC values
            (the reference's correction build takes hours at this size), so
            this case times the apply only (no solve, no parity).
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

HBM = 6458.1  # GB/s, MEASURED_PEAKS.json copy test


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
    b1 = nnz * (2 * 8 + 4) + 8 * (n + 1)
    b2 = nnz * (3 * 8 + 4) + 8 * (n + 1)
    slices = op._plan.m2l_slices if op.far == "fmm" else None
    print(json.dumps({"case": name, "far": op.far, "eps": eps, "fmm_ncrit": ncrit,
                      "m2l_slices": slices, "N": n,
                      "N_over": geom.noversampled, "nnz_per_kind": nnz,
                      "synthetic_corrections": synthetic, "apply_ms": best,
                      "stages_ms": {"far1": st[0], "spmv1": st[1], "far2": st[2],
                                    "spmv2+glue": st[3], "eta": st[4]},
                      "spmv1_GBps": b1 / (st[1] * 1e-3) / 1e9,
                      "spmv2_GBps": b2 / (st[3] * 1e-3) / 1e9,
                      "spmv1_frac_hbm": b1 / (st[1] * 1e-3) / 1e9 / HBM,
                      "spmv2_frac_hbm": b2 / (st[3] * 1e-3) / 1e9 / HBM}), flush=True)
    del op
    torch.cuda.empty_cache()


if __name__ == "__main__":
    only = sys.argv[1:]
    c2 = os.path.join(ROOT, "data", "config2.npz")
    if os.path.exists(c2) and (not only or "config2" in only):
        g = dict(np.load(c2))
        cset = CorrectionSet.from_arrays(g)
        run("config2", g, cset, 1e-10, "direct")
        run("config2", g, cset, 1e-10, "fmm")
    c3 = os.path.join(ROOT, "data", "config3_geom.npz")
    if os.path.exists(c3) and (not only or "config3" in only):
        g = dict(np.load(c3))
        indptr, idx = pattern_from_near(g)
        gen = torch.Generator(device="cuda").manual_seed(3)
        vals = {k: 1e-4 * torch.randn(idx.numel(), dtype=torch.float64, device="cuda",
                                      generator=gen)
                for k in ("s", "sprime", "spp_plus_dprime")}
        cset = CorrectionSet(indptr, idx, vals)
        run("config3", g, cset, 5e-8, "fmm", synthetic=True)
        run("config3", g, cset, 5e-8, "fmm", synthetic=True, ncrit=300, m2l="fp64")
        run("config3", g, cset, 5e-8, "fmm", synthetic=True, ncrit=300)
        run("config3", g, cset, 1e-9, "fmm", synthetic=True, ncrit=300, m2l="fp64")
        run("config3", g, cset, 1e-9, "fmm", synthetic=True, ncrit=300)
        run("config3", g, cset, 5e-8, "direct", reps=2, synthetic=True)
    c4 = os.path.join(ROOT, "data", "config4_geom.npz")
    if os.path.exists(c4) and (not only or "config4" in only):
        g = dict(np.load(c4))
        indptr, idx = pattern_from_near(g)
        gen = torch.Generator(device="cuda").manual_seed(4)
        vals = {k: 1e-4 * torch.randn(idx.numel(), dtype=torch.float64, device="cuda",
                                      generator=gen)
                for k in ("s", "sprime", "spp_plus_dprime")}
        cset = CorrectionSet(indptr, idx, vals)
        del indptr
        torch.cuda.empty_cache()
        run("config4", g, cset, 1e-9, "fmm", reps=2, synthetic=True, ncrit=300)
        run("config4", g, cset, 1e-9, "fmm", reps=2, synthetic=True, ncrit=300, m2l="fp64")
        run("config4", g, cset, 1e-9, "fmm", reps=2, synthetic=True, ncrit=120)
