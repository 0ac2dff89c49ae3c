"""Generate golden fixtures by running the REFERENCE package (lapbel) in this
container.  Test infrastructure only: nothing in the product imports this.

    python scripts/make_golden.py small      # tests/golden/*.npz (committed)
    python scripts/make_golden.py config2    # data/config2.npz (large, git-ignored)

The reference is imported from /root/reference/pkg/src (read-only); numba's
cache is redirected to a writable temp dir.  Every fixture stores its seed and
the reference call that produced it so the tests can say what they pin.
"""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_lapbel")
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from lapbel import fmm, shapes  # noqa: E402
from lapbel._pointsum import run_grouped_direct  # noqa: E402
from lapbel.harmonics import real_ynm  # noqa: E402
from lapbel.kernels import KernelKind  # noqa: E402
from lapbel import operators as ref_operators  # noqa: E402
from lapbel.operators import FORMULATIONS, LayerOperatorSet  # noqa: E402
from lapbel.quadrature import build_near_map, compute_corrections  # noqa: E402
from lapbel.simplex import reference_element, split4  # noqa: E402
from lapbel.solver import SolveConfig, solve_laplace_beltrami, gmres  # noqa: E402
from lapbel.surface import build_from_samples  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "data")

KIND_ORDER = ["s", "d", "sprime", "grads1", "grads2", "grads3",
              "spp_plus_dprime"]


# ---------------------------------------------------------------------------
# geometry generators that the reference lacks (BASELINE configs 1-2)

def icosahedron():
    g = (1.0 + 5 ** 0.5) / 2.0
    v = []
    for a in (-1.0, 1.0):
        for b in (-g, g):
            v += [(0.0, a, b), (a, b, 0.0), (b, 0.0, a)]
    v = np.array(v)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    # faces = triples of mutually adjacent vertices (edge length = min dist)
    d = np.linalg.norm(v[:, None] - v[None], axis=-1)
    e = d[d > 1e-9].min()
    adj = np.abs(d - e) < 1e-9
    faces = []
    for i in range(12):
        for j in range(i + 1, 12):
            if not adj[i, j]:
                continue
            for k in range(j + 1, 12):
                if adj[i, k] and adj[j, k]:
                    f = [i, j, k]
                    nrm = np.cross(v[j] - v[i], v[k] - v[i])
                    if np.dot(nrm, v[i] + v[j] + v[k]) < 0:
                        f = [i, k, j]
                    faces.append(f)
    assert len(faces) == 20
    return v, faces


def icosphere(order: int, nsplit: int = 2):
    """Unit sphere from the radially projected, twice 4-way split icosahedron
    (320 flat triangles for nsplit=2), built through the reference's public
    build_from_samples with the radial-projection chart (the math of
    shapes.py:85-93)."""
    v, faces = icosahedron()
    tris = [np.array([v[a], v[b], v[c]]) for a, b, c in faces]
    for _ in range(nsplit):
        tris = [t for tri in tris for t in split4(tri)]
    ref = reference_element(order)
    uv = ref.nodes
    xs, xus, xvs = [], [], []
    for t in tris:
        e1 = t[1] - t[0]
        e2 = t[2] - t[0]
        c = t[0] + np.outer(uv[:, 0], e1) + np.outer(uv[:, 1], e2)
        r = np.linalg.norm(c, axis=1, keepdims=True)
        x = c / r

        def proj(dc):
            return (dc - x * np.einsum("ik,ik->i", x, dc)[:, None]) / r
        xs.append(x)
        xus.append(proj(np.broadcast_to(e1, c.shape)))
        xvs.append(proj(np.broadcast_to(e2, c.shape)))
    disc = build_from_samples(order, np.array(xs), np.array(xus),
                              np.array(xvs), metadata={"geometry": "icosphere"})
    vol3 = float(np.dot(disc.weights,
                        np.einsum("ik,ik->i", disc.nodes, disc.normals)))
    assert vol3 > 0
    return disc


# ---------------------------------------------------------------------------
# packing helpers

def geometry_arrays(disc, prefix=""):
    ref = reference_element(disc.order)
    return {
        prefix + "order": np.int64(disc.order),
        prefix + "nb": np.int64(disc.nodes_per_patch),
        prefix + "npatches": np.int64(disc.npatches),
        prefix + "nodes": disc.nodes,
        prefix + "normals": disc.normals,
        prefix + "weights": disc.weights,
        prefix + "curvature": disc.curvature,
        prefix + "tangents_u": disc.tangents_u,
        prefix + "tangents_v": disc.tangents_v,
        prefix + "inv_metric": disc.inv_metric,
        prefix + "node_patch": disc.node_patch,
        prefix + "over_nodes": disc.over_nodes,
        prefix + "over_normals": disc.over_normals,
        prefix + "over_weights": disc.over_weights,
        prefix + "over_interp": ref.over_interp,
        # chart coefficients + node preimages + Vandermonde inverse: what the
        # correction build (quadrature.py:159-220, 527-559) consumes
        prefix + "coeffs_x": disc.coeffs_x,
        prefix + "coeffs_dxdu": disc.coeffs_dxdu,
        prefix + "coeffs_dxdv": disc.coeffs_dxdv,
        prefix + "node_uv": disc.node_uv,
        prefix + "vinv": ref.vinv,
    }


def corrections_arrays(corrs, prefix="corr_"):
    """All kinds share one sparsity pattern (quadrature.py:693-700); store it
    once plus one value array per kind."""
    out = {}
    pat = None
    for kind, nc in corrs.items():
        m = nc.matrix.tocsr()
        m.sort_indices()
        if pat is None:
            pat = (m.indptr.astype(np.int64), m.indices.astype(np.int32))
            out[prefix + "indptr"] = pat[0]
            out[prefix + "indices"] = pat[1]
        else:
            assert np.array_equal(pat[0], m.indptr)
            assert np.array_equal(pat[1], m.indices)
        out[prefix + kind.value] = m.data.astype(np.float64)
    return out


def near_arrays(near, prefix="near_"):
    lens = np.array([len(x) for x in near.near], dtype=np.int64)
    return {prefix + "offsets": np.concatenate([[0], np.cumsum(lens)]),
            prefix + "patches": np.concatenate(near.near).astype(np.int32),
            prefix + "eta": np.float64(near.eta)}


def savez(path, **arrs):
    os.makedirs(os.path.dirname(path), exist_ok=True)
    np.savez_compressed(path, **arrs)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


def lists_to_csr(lists):
    lens = np.array([0 if x is None else len(x) for x in lists], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(lens)])
    flat = np.concatenate([np.asarray(x, dtype=np.int64) for x in lists
                           if x is not None and len(x)]) if off[-1] else \
        np.zeros(0, np.int64)
    return off, flat


def cached_opset(disc, form, eps, near, corrs, t_q, use_fmm=False):
    """LayerOperatorSet whose constructor reuses already built corrections
    (compute_corrections is deterministic; rebuilding costs minutes)."""
    orig = ref_operators.compute_corrections

    def cached(d, n, kinds, e):
        return {k: corrs[k] for k in kinds}, t_q
    ref_operators.compute_corrections = cached
    try:
        return LayerOperatorSet(disc, form, eps, use_fmm=use_fmm, near=near)
    finally:
        ref_operators.compute_corrections = orig


# ---------------------------------------------------------------------------
# small fixtures


def gold_p2p():
    """evaluate_direct (fmm.py:215) and run_grouped_direct (_pointsum.py:92)
    on seeded clouds."""
    out = {}
    # case A: test_fmm.py:58-69 cloud (charge-only and dipole-only densities)
    rng = np.random.default_rng(42)
    pos = rng.uniform(0, 1, (3000, 3))
    tgt = rng.uniform(0, 1, (800, 3))
    ch = rng.standard_normal((2, 3000))
    ch[1] = 0
    dip = rng.standard_normal((2, 3000, 3))
    dip[0] = 0
    res = fmm.evaluate_direct(fmm.FmmSources(pos, ch, dip), tgt,
                              ("pot", "grad", "hess"))
    out.update(a_src=pos, a_tgt=tgt, a_ch=ch, a_dip=dip, a_pot=res.pot,
               a_grad=res.grad, a_hess=res.hess)
    # case B: sources == targets on the unit sphere (self pairs skipped),
    # mixed charge+dipole on one density, nd=3, all levels
    rng = np.random.default_rng(105)
    x = rng.standard_normal((700, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    ch = rng.standard_normal((3, 700))
    dip = rng.standard_normal((3, 700, 3))
    ch[2] = 0.0
    dip[0] = 0.0
    res = fmm.evaluate_direct(fmm.FmmSources(x, ch, dip), x,
                              ("pot", "grad", "hess"))
    out.update(b_x=x, b_ch=ch, b_dip=dip, b_pot=res.pot, b_grad=res.grad,
               b_hess=res.hess)
    # case C: grouped direct with irregular groups and an empty group
    rng = np.random.default_rng(7)
    ntf = 300
    t_xyz = rng.uniform(-1, 1, (ntf, 3))
    t_out = rng.permutation(400)[:ntf]
    t_off = np.array([0, 17, 17, 140, 141, 300], dtype=np.int64)
    nsf = 900
    s_xyz = rng.uniform(-1, 1, (nsf, 3))
    s_xyz[:5] = t_xyz[:5]                       # coincident pairs in group 0
    s_off = np.array([0, 100, 350, 350, 600, 900], dtype=np.int64)
    s_c = rng.standard_normal((2, nsf))
    s_v = rng.standard_normal((2, nsf, 3))
    use_c = np.array([True, False])
    use_d = np.array([True, True])
    for lev, want in enumerate(({"pot"}, {"pot", "grad"},
                                {"pot", "grad", "hess"})):
        r = run_grouped_direct(t_xyz, t_out, t_off, s_xyz, s_c, s_v, s_off,
                               use_c, use_d, want, 2, 400)
        for k, v in r.items():
            out[f"c{lev}_{k}"] = v
    out.update(c_t_xyz=t_xyz, c_t_out=t_out, c_t_off=t_off, c_s_xyz=s_xyz,
               c_s_off=s_off, c_s_c=s_c, c_s_v=s_v, c_use_c=use_c,
               c_use_d=use_d)
    savez(os.path.join(GOLD, "p2p_direct.npz"), **out)


def gold_config1():
    """BASELINE config 1: icosphere order 5 (N=4800), sigma ~ N(0,1) seed 1,
    charges w*sigma, evaluate_direct pot+grad at the nodes (no 4 pi)."""
    disc = icosphere(5)
    rng = np.random.default_rng(1)
    sigma = rng.standard_normal(disc.nnodes)
    q = disc.weights * sigma
    res = fmm.evaluate_direct(fmm.FmmSources(disc.nodes, q[None]),
                              disc.nodes, ("pot", "grad"))
    savez(os.path.join(GOLD, "config1.npz"), nodes=disc.nodes,
          weights=disc.weights, sigma=sigma, pot=res.pot, grad=res.grad)


def _opset_fixture(name, disc, eps, seed, fvals, exact_u=None, forms=None):
    """Operator bundle + reference applies/solves with use_fmm=False."""
    forms = forms or ("a1", "a2", "a3")
    near = build_near_map(disc, 2.0)
    kinds = []
    for f in forms:
        kinds += list(FORMULATIONS[f])
    kinds = list(dict.fromkeys(kinds))
    corrs, t_q = compute_corrections(disc, near, kinds, eps)
    out = dict(geometry_arrays(disc))
    out.update(corrections_arrays(corrs))
    out.update(near_arrays(near))
    out["eps"] = np.float64(eps)
    out["seed"] = np.int64(seed)
    rng = np.random.default_rng(seed)
    tau = rng.standard_normal(disc.nnodes)
    out["tau"] = tau
    out["f"] = fvals
    if exact_u is not None:
        out["u_exact"] = exact_u
    for form in forms:
        op = cached_opset(disc, form, eps, near, corrs, t_q)
        out[f"{form}_apply"] = op.apply(tau)
        out[f"{form}_phi0"] = op.phi0
        for kind in FORMULATIONS[form]:
            out[f"{form}_layer_{kind.value}"] = op.apply_layer(kind, tau)
        rep = solve_laplace_beltrami(
            op, fvals, SolveConfig(formulation=form, eps=eps,
                                   eps_gmres=1e-10, max_iter=60))
        out[f"{form}_sigma"] = rep.sigma.values
        out[f"{form}_u"] = rep.u.values
        out[f"{form}_hist"] = np.array(rep.residual_history)
        out[f"{form}_converged"] = np.bool_(rep.converged)
        print(name, form, "iters", rep.n_iter, rep.residual_history[-1])
    out["t_q"] = np.float64(t_q)
    savez(os.path.join(GOLD, f"{name}.npz"), **out)


def gold_torus():
    disc = shapes.build_torus(3, 8, 4, 2.0, 1.0)
    f = np.cos(disc.nodes[:, 2]) + disc.nodes[:, 0]
    _opset_fixture("opset_torus_o3", disc, 1e-6, 12, f, forms=("a3",))


def gold_operators():
    # cube sphere (shapes.py:57), order 3, one refinement: N=288
    disc = shapes.build_sphere(3, 1)
    f = real_ynm(2, 1, disc.nodes)
    _opset_fixture("opset_sphere_o3", disc, 1e-6, 11, f, exact_u=-f / 6.0)
    # standard torus (shapes.py:132): varying curvature, genus 1
    disc = shapes.build_torus(3, 8, 4, 2.0, 1.0)
    rng = np.random.default_rng(12)
    f = np.cos(disc.nodes[:, 2]) + rng.standard_normal(disc.nnodes) * 0.0
    f = f + disc.nodes[:, 0]
    _opset_fixture("opset_torus_o3", disc, 1e-6, 12, f, forms=("a3",))


def gold_gmres():
    """gmres (solver.py:48-103) on a seeded nonsymmetric well-conditioned
    system; the reference has no test for it, so pin by running it."""
    rng = np.random.default_rng(21)
    n = 200
    a = np.eye(n) * 2.0 + rng.standard_normal((n, n)) / np.sqrt(n) * 0.5
    b = rng.standard_normal(n)
    x, hist, conv = gmres(lambda v: a @ v, b, 1e-12, 100)
    # happy-breakdown case: rank-deficient Krylov space (identity operator)
    x2, hist2, conv2 = gmres(lambda v: 3.0 * v, b, 1e-12, 50)
    savez(os.path.join(GOLD, "gmres.npz"), a=a, b=b, x=x,
          hist=np.array(hist), conv=np.bool_(conv), x_id=x2,
          hist_id=np.array(hist2), conv_id=np.bool_(conv2))


def _tree_golden(prefix, spos, tpos, ncrit, buffer, out):
    tree = fmm._build_tree(spos, tpos, ncrit)
    cols, v, u, w, x = fmm._build_lists(tree, buffer)
    out[prefix + "spos"] = spos
    out[prefix + "tpos"] = tpos
    out[prefix + "ncrit"] = np.int64(ncrit)
    out[prefix + "buffer"] = np.int64(buffer)
    out[prefix + "center"] = tree.center
    out[prefix + "half"] = np.float64(tree.half)
    out[prefix + "level"] = tree.level.astype(np.int64)
    out[prefix + "ijk"] = tree.ijk
    out[prefix + "parent"] = tree.parent.astype(np.int64)
    out[prefix + "is_leaf"] = tree.is_leaf
    out[prefix + "nsrc"] = tree.nsrc
    for nm, lst in (("children", tree.children), ("src_idx", tree.src_idx),
                    ("tgt_idx", tree.tgt_idx), ("colleagues", cols),
                    ("vlist", v), ("ulist", u), ("wlist", w), ("xlist", x)):
        off, flat = lists_to_csr(lst)
        out[prefix + nm + "_off"] = off
        out[prefix + nm] = flat


def gold_tree():
    out = {}
    rng = np.random.default_rng(42)
    pos = rng.uniform(0, 1, (3000, 3))
    tgt = rng.uniform(0, 1, (800, 3))
    _tree_golden("u1_", pos, tgt, 120, 1, out)
    _tree_golden("u2_", pos, tgt, 120, 2, out)
    rng = np.random.default_rng(11)
    a = rng.normal(0, 0.01, (1500, 3))
    b = rng.uniform(-1, 1, (1500, 3))
    pos = np.vstack([a, b])
    tgt = np.vstack([rng.normal(0, 0.01, (300, 3)),
                     rng.uniform(-1, 1, (300, 3))])
    _tree_golden("cl_", pos, tgt, 40, 1, out)
    _tree_golden("cl2_", pos, tgt, 40, 2, out)
    rng = np.random.default_rng(105)
    x = rng.standard_normal((20000, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    _tree_golden("sph_", x, x, 120, 1, out)
    savez(os.path.join(GOLD, "fmm_tree.npz"), **out)


def gold_unit_ops():
    """SHA-256 of the reference's unit operators (fmm.py:287-354, 431-481),
    so the device FMM's operators can be checked BIT-identical without
    committing hundreds of MB of matrices."""
    import hashlib
    out = {}

    def h(a):
        a = np.ascontiguousarray(a)
        return hashlib.sha256(a.tobytes()).hexdigest()
    for m, buf in ((5, 1), (8, 1), (10, 1)):
        ops = fmm._unit_operators(m, buf)
        keys = list(ops["m2l_canon"].keys())
        offs = list(ops["offsets"].keys())
        pre = f"s{m}_"
        out[pre + "surf"] = h(ops["surf"])
        out[pre + "pinv_up"] = h(ops["pinv_up"])
        out[pre + "pinv_dn"] = h(ops["pinv_dn"])
        out[pre + "m2m"] = h(np.array(ops["m2m"]))
        out[pre + "l2l"] = h(np.array(ops["l2l"]))
        out[pre + "canon"] = h(np.array([ops["m2l_canon"][k] for k in keys]))
        out[pre + "keys"] = h(np.array(keys, dtype=np.int64))
        out[pre + "offs"] = h(np.array(offs, dtype=np.int64))
        out[pre + "okey"] = h(np.array([keys.index(ops["offsets"][d][0]) for d in offs], dtype=np.int64))
        out[pre + "perm"] = h(np.array([ops["offsets"][d][1] for d in offs], dtype=np.int64))
    for n, buf in ((9, 2), (11, 2)):
        ops = fmm._unit_operators_grid(n, buf)
        keys = list(ops["m2l_canon"].keys())
        offs = list(ops["offsets"].keys())
        pre = f"g{n}_"
        out[pre + "pts"] = h(ops["pts"])
        out[pre + "m2m_1d"] = h(np.array(ops["m2m_1d"]))
        out[pre + "canon"] = h(np.array([ops["m2l_canon"][k] for k in keys]))
        out[pre + "keys"] = h(np.array(keys, dtype=np.int64))
        out[pre + "offs"] = h(np.array(offs, dtype=np.int64))
        out[pre + "okey"] = h(np.array([keys.index(ops["offsets"][d][0]) for d in offs], dtype=np.int64))
        out[pre + "perm"] = h(np.array([ops["offsets"][d][1] for d in offs], dtype=np.int64))
        out[pre + "vinv"] = h(fmm._cheb_vinv(n))
    import json
    path = os.path.join(GOLD, "unit_ops_sha256.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path)


def gold_fmm():
    """FmmPlan.apply outputs (fmm.py:784) for the test_fmm cloud at the three
    representation regimes, to pin the GPU FMM against the SAME approximation
    (not only against the direct sum)."""
    out = {}
    rng = np.random.default_rng(42)
    pos = rng.uniform(0, 1, (3000, 3))
    tgt = rng.uniform(0, 1, (800, 3))
    ch = rng.standard_normal((2, 3000))
    ch[1] = 0
    dip = rng.standard_normal((2, 3000, 3))
    dip[0] = 0
    out.update(src=pos, tgt=tgt, ch=ch, dip=dip)
    for eps in (1e-3, 1e-6, 1e-9):
        src = fmm.FmmSources(pos, ch, dip)
        res = fmm.evaluate_fmm(src, tgt, eps, ("pot", "grad", "hess"))
        key = f"e{int(round(-np.log10(eps)))}_"
        out[key + "pot"] = res.pot
        out[key + "grad"] = res.grad
        out[key + "hess"] = res.hess
    # clustered cloud, ncrit 40, charge only (test_fmm.py:114-125)
    rng = np.random.default_rng(11)
    a = rng.normal(0, 0.01, (1500, 3))
    b = rng.uniform(-1, 1, (1500, 3))
    pos = np.vstack([a, b])
    tgt = np.vstack([rng.normal(0, 0.01, (300, 3)),
                     rng.uniform(-1, 1, (300, 3))])
    ch = rng.standard_normal((1, 3000))
    res = fmm.evaluate_fmm(fmm.FmmSources(pos, ch), tgt, 1e-6,
                           ("pot", "grad"), ncrit=40)
    out.update(cl_src=pos, cl_tgt=tgt, cl_ch=ch, cl_pot=res.pot,
               cl_grad=res.grad)
    savez(os.path.join(GOLD, "fmm_apply.npz"), **out)


# ---------------------------------------------------------------------------
# large bundle (git-ignored): BASELINE config 2


def config2(eps=1e-10):
    t0 = time.time()
    disc = icosphere(7)
    print("config2 N", disc.nnodes, "Nover", disc.noversampled)
    near = build_near_map(disc, 2.0)
    kinds = [KernelKind.SINGLE_LAYER, KernelKind.DOUBLE_LAYER,
             KernelKind.SPRIME, KernelKind.SPP_PLUS_DPRIME]
    corrs, t_q = compute_corrections(disc, near, kinds, eps)
    print("t_q", t_q)
    out = dict(geometry_arrays(disc))
    out.update(corrections_arrays(corrs))
    out.update(near_arrays(near))
    out["eps"] = np.float64(eps)
    out["t_q"] = np.float64(t_q)
    f = real_ynm(3, 2, disc.nodes)
    out["f"] = f
    out["u_exact"] = -f / 12.0
    rng = np.random.default_rng(2)
    tau = rng.standard_normal(disc.nnodes)
    out["tau"] = tau
    savez(os.path.join(DATA, "config2.npz"), **out)   # checkpoint
    for form in ("a3", "a2"):
        op = cached_opset(disc, form, eps, near, corrs, t_q)
        t1 = time.time()
        out[f"{form}_apply"] = op.apply(tau)
        out[f"{form}_t_apply"] = np.float64(time.time() - t1)
        rep = solve_laplace_beltrami(
            op, f, SolveConfig(formulation=form, eps=eps, eps_gmres=1e-10))
        out[f"{form}_sigma"] = rep.sigma.values
        out[f"{form}_u"] = rep.u.values
        out[f"{form}_hist"] = np.array(rep.residual_history)
        out[f"{form}_t_s"] = np.float64(rep.t_s)
        print(form, rep.n_iter, rep.residual_history, rep.t_s)
        savez(os.path.join(DATA, "config2.npz"), **out)
    print("total", time.time() - t0)


def config2_geom():
    """tests/golden/config2_geom.npz (committed): data/config2.npz without the
    corrections (the bench's fallback builds them on the device) but with the
    reference's A3 apply of the seeded tau and its A3 solve, so the parity
    spot checks stay reference-anchored."""
    z = np.load(os.path.join(DATA, "config2.npz"))
    keep = {k: z[k] for k in z.files if not k.startswith("corr_")
            and not k.startswith("a2_")}
    savez(os.path.join(GOLD, "config2_geom.npz"), **keep)


def config3():
    """BASELINE config 3 geometry (build_torus(7, 64, 32, 2, 1): N = 114,688)
    and its near map (eta 2, cap raised to 256: the default 128 raises
    NearMapCapError here).  Corrections are NOT built (the reference's t_q is
    hours at this size): timing runs put synthetic values on this exact
    sparsity pattern and say so."""
    t0 = time.time()
    disc = shapes.build_torus(7, 64, 32, 2.0, 1.0)
    near = build_near_map(disc, 2.0, cap=256)
    out = dict(geometry_arrays(disc))
    out.update(near_arrays(near))
    savez(os.path.join(DATA, "config3_geom.npz"), **out)
    print("config3", disc.nnodes, disc.noversampled, time.time() - t0)


def wavy_torus(order=9, nu=82, nv=163):
    """BASELINE config 4 surface: tube radius r(theta, phi) = 1 + 0.25 cos(5 phi)
    sin(3 theta) around the R = 2 torus; theta poloidal (u axis), phi toroidal
    (v axis), triangles from the reference's own parameter grid with the
    outward (flip=True) orientation (shapes.py:106-129), sampled with its
    _sample_patches and built through build_from_samples (surface.py:310)."""
    def chart(p):
        th, ph = p[:, 0], p[:, 1]
        rho = 1.0 + 0.25 * np.cos(5 * ph) * np.sin(3 * th)
        rho_t = 0.75 * np.cos(5 * ph) * np.cos(3 * th)
        rho_p = -1.25 * np.sin(5 * ph) * np.sin(3 * th)
        er = np.column_stack([np.cos(ph), np.sin(ph), np.zeros_like(ph)])
        ep = np.column_stack([-np.sin(ph), np.cos(ph), np.zeros_like(ph)])
        ez = np.array([0.0, 0.0, 1.0])[None, :]
        ring = 2.0 + rho * np.cos(th)
        x = ring[:, None] * er + (rho * np.sin(th))[:, None] * ez
        xt = (rho_t * np.cos(th) - rho * np.sin(th))[:, None] * er \
            + (rho_t * np.sin(th) + rho * np.cos(th))[:, None] * ez
        xp = (rho_p * np.cos(th))[:, None] * er + ring[:, None] * ep \
            + (rho_p * np.sin(th))[:, None] * ez
        return x, xt, xp
    xs, xus, xvs = shapes._sample_patches(
        order, shapes._param_grid_triangles(nu, nv, flip=True), chart)
    disc = build_from_samples(order, xs, xus, xvs,
                              metadata={"geometry": "wavy-torus", "nu": nu, "nv": nv})
    shapes._check_outward(disc, "wavy-torus")
    return disc


def config4():
    """BASELINE config 4 geometry (N = 1,202,940 at reference order 9) and its
    near map (eta 2).  Corrections are not built (a day of reference CPU
    time); timing runs put synthetic values on this pattern.  A1-only arrays
    are dropped to keep the file small."""
    t0 = time.time()
    disc = wavy_torus()
    print("config4 geometry", disc.nnodes, disc.noversampled, time.time() - t0, flush=True)
    near = build_near_map(disc, 2.0, cap=256)
    print("near map", time.time() - t0, flush=True)
    out = {k: v for k, v in geometry_arrays(disc).items()
           if k not in ("tangents_u", "tangents_v", "inv_metric")}
    out.update(near_arrays(near))
    savez(os.path.join(DATA, "config4_geom.npz"), **out)
    print("config4", time.time() - t0)


def augment():
    """Add the correction-build inputs (chart coefficients, node preimages,
    vinv) to fixtures generated before geometry_arrays carried them, by
    rebuilding the same deterministic geometry (no correction rebuild)."""
    cases = [
        (os.path.join(GOLD, "opset_sphere_o3.npz"), lambda: shapes.build_sphere(3, 1)),
        (os.path.join(GOLD, "opset_torus_o3.npz"), lambda: shapes.build_torus(3, 8, 4, 2.0, 1.0)),
        (os.path.join(DATA, "config2.npz"), lambda: icosphere(7)),
        (os.path.join(DATA, "config3_geom.npz"), lambda: shapes.build_torus(7, 64, 32, 2.0, 1.0)),
    ]
    for path, make in cases:
        if not os.path.exists(path):
            continue
        old = dict(np.load(path))
        disc = make()
        assert np.array_equal(old["nodes"], disc.nodes), path
        new = geometry_arrays(disc)
        for k in ("coeffs_x", "coeffs_dxdu", "coeffs_dxdv", "node_uv", "vinv"):
            old[k] = new[k]
        savez(path, **old)


def gold_quad():
    """Correction-build goldens (quadrature.py:663-701): the reference's
    near map and corrections for the non-PV kinds (S, D, S', S''+D') on an
    order-7 cube sphere (N = 336) at eps 1e-10 (the order-3 sphere/torus
    opset fixtures and data/config2.npz cover the other cases)."""
    kinds = [KernelKind.SINGLE_LAYER, KernelKind.DOUBLE_LAYER,
             KernelKind.SPRIME, KernelKind.SPP_PLUS_DPRIME]
    cases = (("quad_sphere_o7", shapes.build_sphere(7, 0), 1e-10),)
    if len(sys.argv) > 2:  # e.g. `gold_quad o9`: the order-9 cube sphere (config 4's order)
        cases = (("quad_sphere_o9", shapes.build_sphere(9, 0), 1e-9),)
    for name, disc, eps in cases:
        near = build_near_map(disc, 2.0)
        corrs, t_q = compute_corrections(disc, near, kinds, eps)
        out = dict(geometry_arrays(disc))
        out.update(corrections_arrays(corrs))
        out.update(near_arrays(near))
        out["eps"] = np.float64(eps)
        out["t_q"] = np.float64(t_q)
        print(name, disc.nnodes, "t_q", t_q)
        savez(os.path.join(GOLD, f"{name}.npz"), **out)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        gold_p2p()
        gold_config1()
        gold_gmres()
        gold_tree()
        gold_fmm()
        gold_operators()
    elif what == "config2":
        config2()
    else:
        globals()[what]()
