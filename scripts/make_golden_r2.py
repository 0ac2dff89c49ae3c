"""Round-2 golden fixtures: pins of the BASELINE-scale configs (3, 4, 5) and
the config-2 A2 solve to the REFERENCE package (lapbel), run in this
container.  Test infrastructure only: nothing in the product imports this.

    python scripts/make_golden_r2.py config5_tree   # tests/golden/config5_tree_sha256.json
    python scripts/make_golden_r2.py config5_fmm    # tests/golden/config5_fmm_1e6.npz
    python scripts/make_golden_r2.py config3_rows   # tests/golden/config3_rows.npz
    python scripts/make_golden_r2.py config4_rows   # tests/golden/config4_rows.npz
    python scripts/make_golden_r2.py hodge_small    # tests/golden/hodge_torus_o7.npz
    python scripts/make_golden_r2.py config2_a2     # tests/golden/config2_ref.npz

Row-sampled corrections follow SURVEY §7: a NearMap (quadrature.py:66-73)
whose `near` lists are empty except for the sampled targets, passed to
compute_corrections (quadrature.py:663-701); the sampled rows are
bit-identical to the full build's (validated in the survey), at a cost of
seconds instead of hours.  Large structures (the 10^6-point octree and
lists, full near maps) are committed as SHA-256 digests of their canonical
int64/fp64 bytes, so the device build is checked bit-exact without
committing hundreds of MB.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as mg  # noqa: E402  (sets NUMBA_CACHE_DIR and the reference path)

import numpy as np  # noqa: E402

from lapbel import fmm, shapes  # noqa: E402
from lapbel.hodge import TangentialField, hodge_decompose  # noqa: E402
from lapbel.kernels import KernelKind  # noqa: E402
from lapbel.quadrature import NearMap, build_near_map, compute_corrections  # noqa: E402
from lapbel.solver import SolveConfig  # noqa: E402

GOLD = mg.GOLD
A3_KINDS = [KernelKind.SINGLE_LAYER, KernelKind.SPRIME, KernelKind.SPP_PLUS_DPRIME]


def sha(a, dtype=None):
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return hashlib.sha256(a.tobytes()).hexdigest()


def cloud(n, seed=105):
    """BASELINE config 5 point cloud: seeded standard normals normalised onto
    the unit sphere (seed 100 + config)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x


# ---------------------------------------------------------------------------
# config 5: octree + lists at 10^6 (fmm.py:559-715), reference FMM at 10^6


def tree_digests(spos, tpos, ncrit, buffer):
    t0 = time.time()
    tree = fmm._build_tree(spos, tpos, ncrit)
    t1 = time.time()
    cols, v, u, w, x = fmm._build_lists(tree, buffer)
    t2 = time.time()
    out = {"ncrit": ncrit, "buffer": buffer, "nbox": int(len(tree.level)),
           "nleaf": int(np.sum(tree.is_leaf)), "t_tree_s": t1 - t0,
           "t_lists_s": t2 - t1,
           "center": sha(tree.center, np.float64), "half": float(tree.half),
           "level": sha(tree.level, np.int64), "ijk": sha(tree.ijk, np.int64),
           "parent": sha(tree.parent, np.int64), "nsrc": sha(tree.nsrc, np.int64),
           "is_leaf": sha(tree.is_leaf, np.bool_)}
    for nm, lst in (("children", tree.children), ("src_idx", tree.src_idx),
                    ("tgt_idx", tree.tgt_idx), ("colleagues", cols),
                    ("vlist", v), ("ulist", u), ("wlist", w), ("xlist", x)):
        off, flat = mg.lists_to_csr(lst)
        out[nm + "_off"] = sha(off, np.int64)
        out[nm] = sha(flat, np.int64)
        out[nm + "_len"] = int(off[-1])
    return out


def config5_tree(n=1_000_000):
    x = cloud(n)
    res = {"n": n, "seed": 105, "cloud": "default_rng(105).standard_normal((n,3)) "
           "normalised; sources = targets",
           "x_sha": sha(x, np.float64)}
    for buf in (1, 2):
        d = tree_digests(x, x, 120, buf)
        print("buffer", buf, {k: d[k] for k in ("nbox", "nleaf", "t_tree_s", "t_lists_s",
                                                  "vlist_len", "ulist_len")}, flush=True)
        res[f"b{buf}"] = d
    path = os.path.join(GOLD, "config5_tree_sha256.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)
    print("wrote", path)


def config5_fmm(n=1_000_000, eps=1e-6, nsample=200):
    """FmmPlan(x, x, eps).apply(q, None, ("pot", "grad")) at 10^6 (fmm.py:729,
    784) with the outputs kept at `nsample` seeded target indices, plus the
    exact direct sum at those targets (evaluate_direct, self excluded by
    r = 0) -- the check cli.py:307-314 runs."""
    x = cloud(n)
    q = np.random.default_rng(5).standard_normal((1, n))
    idx = np.sort(np.random.default_rng(205).choice(n, nsample, replace=False))
    t0 = time.time()
    plan = fmm.FmmPlan(x, x, eps)
    t1 = time.time()
    res = plan.apply(q, None, ("pot", "grad"))
    t2 = time.time()
    d = fmm.evaluate_direct(fmm.FmmSources(x, q), x[idx], ("pot", "grad"))
    tag = f"e{int(round(-np.log10(eps)))}_"
    path = os.path.join(GOLD, "config5_fmm_1e6.npz")
    old = dict(np.load(path)) if os.path.exists(path) else {}
    old.update({"n": np.int64(n), "idx": idx, "q_seed": np.int64(5),
                tag + "eps": np.float64(eps), tag + "pot": res.pot[:, idx],
                tag + "grad": res.grad[:, idx], tag + "direct_pot": d.pot,
                tag + "direct_grad": d.grad, tag + "t_plan_s": np.float64(t1 - t0),
                tag + "t_apply_s": np.float64(t2 - t1)})
    mg.savez(path, **old)
    err = np.abs(res.pot[0, idx] - d.pot[0]).max() / np.abs(d.pot).max()
    print("config5 fmm", eps, "plan", t1 - t0, "apply", t2 - t1, "err vs direct", err)


# ---------------------------------------------------------------------------
# configs 3 / 4: row-sampled reference corrections


def sampled_rows(disc, near_full, kinds, eps, targets):
    """compute_corrections on a NearMap holding near lists only for
    `targets`: the rows of those targets exactly as the full
    build would produce them."""
    n = disc.nnodes
    near = [np.zeros(0, np.int64) for _ in range(n)]
    for t in targets:
        near[t] = near_full.near[t]
    inverse = [[] for _ in range(disc.npatches)]
    for t in targets:
        for p in near[t]:
            inverse[p].append(t)
    inverse = [np.array(v, dtype=np.int64) for v in inverse]
    nm = NearMap(eta=near_full.eta, cap=near_full.cap, near=near, inverse=inverse)
    corrs, t_q = compute_corrections(disc, nm, kinds, eps)
    out = {}
    m0 = corrs[kinds[0]].matrix
    off = [0]
    cols = []
    for t in targets:
        a, b = m0.indptr[t], m0.indptr[t + 1]
        cols.append(m0.indices[a:b])
        off.append(off[-1] + (b - a))
    out["rows_off"] = np.array(off, dtype=np.int64)
    out["rows_cols"] = np.concatenate(cols).astype(np.int32)
    for k in kinds:
        m = corrs[k].matrix
        assert np.array_equal(m.indptr[np.asarray(targets) + 1] - m.indptr[np.asarray(targets)],
                              np.diff(out["rows_off"]))
        out["rows_" + k.value] = np.concatenate(
            [m.data[m.indptr[t]:m.indptr[t + 1]] for t in targets])
    return out, t_q


def near_digest(near):
    off, flat = mg.lists_to_csr(near.near)
    return {"near_off_sha": sha(off, np.int64), "near_patches_sha": sha(flat, np.int32),
            "near_total": np.int64(off[-1])}


def _rows_fixture(name, disc, near, kinds, eps, ntarget, seed, extra=None):
    rng = np.random.default_rng(seed)
    targets = np.sort(rng.choice(disc.nnodes, ntarget - 2, replace=False))
    targets = np.unique(np.concatenate([[0, disc.nnodes - 1], targets]))
    rows, t_q = sampled_rows(disc, near, kinds, eps, targets)
    out = {"targets": targets.astype(np.int64), "eps": np.float64(eps),
           "eta": np.float64(near.eta), "cap": np.int64(near.cap),
           "order": np.int64(disc.order), "npatches": np.int64(disc.npatches),
           "nnodes": np.int64(disc.nnodes), "t_q_sample_s": np.float64(t_q),
           "nodes_at": disc.nodes[targets], "normals_at": disc.normals[targets],
           "weights_at": disc.weights[targets], "curvature_at": disc.curvature[targets],
           "area": np.float64(disc.weights.sum()),
           "over_weights_sum": np.float64(disc.over_weights.sum())}
    out.update(near_digest(near))
    out["near_at_off"], out["near_at"] = mg.lists_to_csr([near.near[t] for t in targets])
    out.update(rows)
    out.update(extra or {})
    mg.savez(os.path.join(GOLD, f"{name}.npz"), **out)
    print(name, "targets", len(targets), "t_q(sample)", t_q, flush=True)


def config3_rows(eps=5e-8):
    t0 = time.time()
    disc = shapes.build_torus(7, 64, 32, 2.0, 1.0)
    near = build_near_map(disc, 2.0, cap=256)
    print("config3 geometry + near", time.time() - t0, flush=True)
    _rows_fixture("config3_rows", disc, near, A3_KINDS, eps, 64, 303,
                  {"geometry": np.str_("build_torus(7, 64, 32, 2.0, 1.0)")})


def config4_rows(eps=1e-9):
    t0 = time.time()
    disc = mg.wavy_torus()
    print("config4 geometry", disc.nnodes, time.time() - t0, flush=True)
    near = build_near_map(disc, 2.0, cap=256)
    print("config4 near", time.time() - t0, flush=True)
    _rows_fixture("config4_rows", disc, near, A3_KINDS, eps, 48, 404,
                  {"geometry": np.str_("wavy torus, make_golden.wavy_torus(9, 82, 163)")})


# ---------------------------------------------------------------------------
# config 3's workload (two LB solves of a Hodge decomposition), reference-
# pinned on a reduced torus where the reference's own corrections are cheap


def gaussian_field(nodes, normals, seed_amp, seed_cen, k=16, width=0.5):
    """BASELINE config 3 field: tangential projection (hodge.py:47-54) of
    sum_k a_k exp(-|x - c_k|^2 / (2 width^2)), a_k ~ N(0,1)^3 from
    default_rng(seed_amp), centres c_k = nodes picked by default_rng(seed_cen)."""
    cen = nodes[np.random.default_rng(seed_cen).choice(len(nodes), k, replace=False)]
    amp = np.random.default_rng(seed_amp).standard_normal((k, 3))
    d2 = ((nodes[:, None, :] - cen[None, :, :]) ** 2).sum(-1)
    return np.exp(-d2 / (2 * width ** 2)) @ amp


def hodge_small(eps=1e-10, eps_gmres=1e-10):
    t0 = time.time()
    disc = shapes.build_torus(7, 12, 6, 2.0, 1.0)
    near = build_near_map(disc, 2.0, cap=256)
    corrs, t_q = compute_corrections(disc, near, A3_KINDS, eps)
    print("hodge_small N", disc.nnodes, "t_q", t_q, flush=True)
    op = mg.cached_opset(disc, "a3", eps, near, corrs, t_q, use_fmm=False)
    v = gaussian_field(disc.nodes, disc.normals, 3, 103)
    field = TangentialField.project(disc, v)
    cfg = SolveConfig(formulation="a3", eps=eps, eps_gmres=eps_gmres, max_iter=100)
    res = hodge_decompose(op, field, cfg)
    out = dict(mg.geometry_arrays(disc))
    out.update(mg.near_arrays(near))
    out.update({"eps": np.float64(eps), "eps_gmres": np.float64(eps_gmres),
                "t_q": np.float64(t_q), "field_v": v, "field": field.values,
                "alpha": res.alpha.values, "beta": res.beta.values,
                "grad_alpha": res.grad_alpha.values, "rot_beta": res.rot_beta.values,
                "harmonic": res.harmonic.values, "div_h_norm": np.float64(res.div_h_norm),
                "div_nxh_norm": np.float64(res.div_nxh_norm),
                "n_iter": np.array(res.n_iter, dtype=np.int64),
                "hist_a": np.array(res.reports[0].residual_history),
                "hist_b": np.array(res.reports[1].residual_history),
                "sigma_a": res.reports[0].sigma.values,
                "sigma_b": res.reports[1].sigma.values,
                "metric": disc.metric, "sqrt_det_g": disc.sqrt_det_g})
    mg.savez(os.path.join(GOLD, "hodge_torus_o7.npz"), **out)
    print("hodge_small", res.n_iter, res.div_h_norm, res.div_nxh_norm, time.time() - t0)


# ---------------------------------------------------------------------------
# config 2: the reference's A2 solve + sampled rows of its 4-kind corrections


def config2_a2():
    path = os.path.join(mg.DATA, "config2.npz")
    if not os.path.exists(path) or "a2_u" not in np.load(path).files:
        mg.config2()
    z = np.load(path)
    rng = np.random.default_rng(202)
    n = int(z["nodes"].shape[0])
    targets = np.unique(np.concatenate([[0, n - 1], rng.choice(n, 62, replace=False)]))
    ip, ix = z["corr_indptr"], z["corr_indices"]
    off = [0]
    cols = []
    for t in targets:
        cols.append(ix[ip[t]:ip[t + 1]])
        off.append(off[-1] + ip[t + 1] - ip[t])
    out = {"targets": targets.astype(np.int64), "rows_off": np.array(off, np.int64),
           "rows_cols": np.concatenate(cols).astype(np.int32), "eps": z["eps"]}
    for k in ("s", "d", "sprime", "spp_plus_dprime"):
        v = z["corr_" + k]
        out["rows_" + k] = np.concatenate([v[ip[t]:ip[t + 1]] for t in targets])
    for k in z.files:
        if k.startswith(("a2_", "a3_")):
            out[k] = z[k]
    mg.savez(os.path.join(GOLD, "config2_ref.npz"), **out)



def geom_coeffs():
    """SHA-256 of the chart coefficients the reference's own generators hand
    to build_from_coefficients (surface.py:317-320) for the BASELINE
    geometries: configs 1-2 (icosphere, orders 5/7), 3 (build_torus(7, 64,
    32, 2, 1)) and 4 (the wavy torus, order 9) -- the device geometry build
    (paper_2111_10743_b200/shapes.py) must start from identical bytes."""
    from lapbel.simplex import reference_element as rref
    cap = {}

    class _Stop(Exception):
        pass

    def grab(order, x, xu, xv, **kw):
        v = rref(order).vinv
        cap["c"] = [np.einsum("ij,pjc->pic", v, np.asarray(a)) for a in (x, xu, xv)]
        raise _Stop
    shapes.build_from_samples = grab
    mg.build_from_samples = grab
    out = {}
    for name, f in (("icosphere_o5", lambda: mg.icosphere(5)),
                    ("icosphere_o7", lambda: mg.icosphere(7)),
                    ("torus_o7_64x32", lambda: shapes.build_torus(7, 64, 32, 2.0, 1.0)),
                    ("torus_o7_12x6", lambda: shapes.build_torus(7, 12, 6, 2.0, 1.0)),
                    ("wavy_o9_82x163", lambda: mg.wavy_torus())):
        try:
            f()
        except _Stop:
            pass
        out[name] = {k: sha(a, np.float64) for k, a in zip(("x", "dxdu", "dxdv"), cap["c"])}
        out[name]["npatches"] = int(cap["c"][0].shape[0])
    path = os.path.join(GOLD, "geom_coeffs_sha256.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    for what in sys.argv[1:]:
        t0 = time.time()
        globals()[what]()
        print(f"== {what} done in {time.time() - t0:.1f} s", flush=True)
