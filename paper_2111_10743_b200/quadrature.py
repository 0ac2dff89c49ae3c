"""Near-correction build on the B200.

Mirror of lapbel.quadrature's public operations for the kinds the A2/A3
formulations use: ``build_near_map`` (quadrature.py:76-104) and
``compute_corrections`` (quadrature.py:663-701) for all seven kinds.
The reference runs them once per geometry on the CPU (t_q: 438 s at BASELINE
config 2, hours at config 3); here the near map is one device pass over the
patch bounding spheres and the adaptive singular quadrature runs one CTA per
(target, patch) pair (``csrc/quad.cu``); the gradient kinds (A1) add the
principal-value constants (quadrature.py:562-590): the adaptive curvature and
double-layer compensation integrals on the same kernel and the boundary line
integral as one warp per (target, edge).

Host work here is the reference's own small precomputations restated (leaf
rules, k-major permutation, patch bounding spheres), so the device receives
the same numbers the reference's kernels see.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .operators import KIND_CODE, CorrectionSet, KernelKind, as_kind

__all__ = ["NearMap", "NearMapCapError", "AdaptiveDepthError", "build_near_map",
           "compute_corrections", "build_correction_set", "patch_bounds",
           "leaf_rules", "kmajor_permutation"]

GRAD_KINDS = (KernelKind.GRAD_S1, KernelKind.GRAD_S2, KernelKind.GRAD_S3)

# host / device split of the last build_correction_set call (seconds)
LAST_BUILD: dict = {}


NearMapCapError = _lib.NearMapCapError        # quadrature.py:58-59
AdaptiveDepthError = _lib.AdaptiveDepthError  # quadrature.py:62-63


@dataclass
class NearMap:
    """Per-target near patches (self first) as one flat list: patches of
    target t are ``patches[offsets[t]:offsets[t + 1]]`` (quadrature.py:66-73
    keeps a list of arrays; ``near`` / ``inverse`` rebuild that view)."""

    eta: float
    cap: int
    offsets: np.ndarray   # (N + 1,) int64
    patches: np.ndarray   # (nnz,) int32

    @property
    def near(self):
        return [self.patches[self.offsets[t]:self.offsets[t + 1]].astype(np.int64)
                for t in range(len(self.offsets) - 1)]

    @property
    def inverse(self):
        npat = int(self.patches.max()) + 1 if len(self.patches) else 0
        tg = np.repeat(np.arange(len(self.offsets) - 1), np.diff(self.offsets))
        order = np.argsort(self.patches, kind="stable")
        cuts = np.searchsorted(self.patches[order], np.arange(npat + 1))
        return [tg[order[cuts[p]:cuts[p + 1]]] for p in range(npat)]


# ---------------------------------------------------------------------------
# host precomputations (restated from the reference)


def patch_bounds(disc):
    """Patch bounding spheres over nodes + oversampled nodes
    (surface.py:146-153, same numpy operations)."""
    nb = disc.nodes_per_patch
    npat = disc.npatches
    pos = np.asarray(disc.nodes).reshape(npat, nb, 3)
    over = np.asarray(disc.over_nodes).reshape(npat, -1, 3)
    allpts = np.concatenate([pos, over], axis=1)
    centers = allpts.mean(axis=1)
    radii = np.sqrt(((allpts - centers[:, None, :]) ** 2).sum(-1)).max(axis=1)
    return centers, radii


def kmajor_permutation(order):
    """deg-major column j <- k-major column perm[j] (quadrature.py:147-156)."""
    perm = np.empty(order * (order + 1) // 2, dtype=np.int64)
    j = 0
    for d in range(order):
        for k in range(d + 1):
            l = d - k
            perm[j] = k * order - k * (k - 1) // 2 + l
            j += 1
    return perm


def koornwinder_norms_kmajor(order):
    """sqrt(2(2k+1)(k+l+1)) per k-major column (_leafeval.py:56)."""
    return np.array([np.sqrt(2.0 * (2 * k + 1) * (k + l + 1))
                     for k in range(order) for l in range(order - k)])


def leaf_rules(order):
    """Smooth leaf rule triangle_rule(p + 2) (simplex.py:134-150) and the
    Duffy rule concentrated at vertex 0 (quadrature.py:181-190), each as
    (nq, 3) rows of (u or a, v or b, weight)."""
    from scipy.special import roots_jacobi, roots_legendre
    n = order + 2
    xa, wa = roots_legendre(n)
    xb, wb = roots_jacobi(n, 1.0, 0.0)
    A, B = np.meshgrid(xa, xb, indexing="ij")
    WA, WB = np.meshgrid(wa, wb, indexing="ij")
    v = (1.0 + B) / 2.0
    u = (1.0 + A) * (1.0 - B) / 4.0
    w = WA * WB / 8.0
    srule = np.column_stack([u.ravel(), v.ravel(), w.ravel()])
    ga, gwa = roots_legendre(order + 2)
    gb, gwb = roots_legendre(order + 1)
    a = 0.5 * (ga + 1.0)
    b = 0.5 * (gb + 1.0)
    A, B = np.meshgrid(a, b, indexing="ij")
    WA, WB = np.meshgrid(gwa * 0.5, gwb * 0.5, indexing="ij")
    drule = np.column_stack([A.ravel(), B.ravel(), (WA * WB * A).ravel()])
    return srule, drule


def _bind():
    L = _lib.load()
    return L


def _dev(a):
    """numpy -> contiguous CUDA tensor of the SAME dtype (_lib.to_device
    converts to float64)."""
    t = _lib.torch()
    _lib.require_cuda()
    return t.from_numpy(np.ascontiguousarray(a)).to("cuda")


# ---------------------------------------------------------------------------
# near map


def build_near_map(disc, eta: float = 2.0, cap: int = 128) -> NearMap:
    """Near(x_i) = patches whose bounding sphere is within eta radii of x_i,
    plus always the self patch (quadrature.py:76-104), on the device."""
    if eta <= 0:
        raise ValueError("eta must be positive")
    t = _lib.torch()
    _lib.require_cuda()
    L = _bind()
    centers, radii = patch_bounds(disc)
    rad = (1.0 + eta) * radii
    n = disc.nnodes
    nodes = _dev(np.asarray(disc.nodes, dtype=float))
    cen = _dev(np.asarray(centers, dtype=float))
    rd = _dev(np.asarray(rad, dtype=float))
    npat = _dev(np.asarray(disc.node_patch, dtype=np.int64))
    counts = t.empty(n, dtype=t.int32, device="cuda")
    stream = _lib.stream_handle(None)
    _lib.check(L.lb_near_map_count(_lib.ptr(nodes), n, _lib.ptr(cen), _lib.ptr(rd),
                                   centers.shape[0], _lib.ptr(npat), _lib.ptr(counts),
                                   stream), "lb_near_map_count")
    offsets = t.zeros(n + 1, dtype=t.int64, device="cuda")
    offsets[1:] = t.cumsum(counts.to(t.int64), 0)
    cmax = int(counts.max()) if n else 0
    if cmax > cap:
        tt = int(t.argmax(counts))
        raise NearMapCapError(
            f"target {tt} has {cmax} near patches (cap {cap}); "
            "the mesh is under-resolved for eta = {:.2f}".format(eta))
    patches = t.empty(int(offsets[-1]), dtype=t.int32, device="cuda")
    _lib.check(L.lb_near_map_fill(_lib.ptr(nodes), n, _lib.ptr(cen), _lib.ptr(rd),
                                  centers.shape[0], _lib.ptr(npat), _lib.ptr(offsets),
                                  _lib.ptr(patches), stream), "lb_near_map_fill")
    return NearMap(eta=float(eta), cap=int(cap), offsets=offsets.cpu().numpy(),
                   patches=patches.cpu().numpy())


# ---------------------------------------------------------------------------
# corrections


class _Desc(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int), ("nk", ctypes.c_int),
                ("kinds", ctypes.c_int * 7), ("eps", ctypes.c_double),
                ("coeffs_km", ctypes.c_void_p), ("nodes", ctypes.c_void_p),
                ("normals", ctypes.c_void_p), ("node_uv", ctypes.c_void_p),
                ("node_patch", ctypes.c_void_p), ("pair_tgt", ctypes.c_void_p),
                ("pair_pat", ctypes.c_void_p), ("pair_pos", ctypes.c_void_p),
                ("npairs", ctypes.c_int64), ("srule", ctypes.c_void_p),
                ("nqs", ctypes.c_int), ("drule", ctypes.c_void_p),
                ("nqd", ctypes.c_int), ("knorm", ctypes.c_void_p),
                ("kmajor_perm", ctypes.c_void_p), ("vinv", ctypes.c_void_p),
                ("over_interp", ctypes.c_void_p), ("nbo", ctypes.c_int),
                ("over_nodes", ctypes.c_void_p), ("over_normals", ctypes.c_void_p),
                ("over_weights", ctypes.c_void_p), ("values", ctypes.c_void_p * 7),
                ("stats", ctypes.c_void_p), ("n", ctypes.c_int64),
                ("hcoeff_km", ctypes.c_void_p), ("gauss", ctypes.c_void_p),
                ("ng", ctypes.c_int)]


def _require(disc, name):
    v = getattr(disc, name, None)
    if v is None:
        raise ValueError(f"the correction build needs disc.{name} "
                         "(SurfaceDiscretization field)")
    return np.asarray(v)


def _vinv(disc):
    v = getattr(disc, "vinv", None)
    if v is not None:
        return np.asarray(v, dtype=float)
    # ReferenceElement.vinv (simplex.py:359-383), restated in simplex.py
    from .simplex import reference_element
    return reference_element(disc.order).vinv


def build_correction_set(disc, near: NearMap, kinds, eps: float):
    """Device correction build -> (CorrectionSet on the device, t_q seconds).
    The pattern is the reference's CSR pattern (rows = targets, nb columns per
    near patch, sorted, quadrature.py:691-700); values per kind."""
    if not (1e-12 <= eps <= 1e-3):
        raise ValueError("eps must lie in [1e-12, 1e-3]")
    kinds = [as_kind(k) for k in kinds]
    want_pv = any(k in GRAD_KINDS for k in kinds)
    t = _lib.torch()
    _lib.require_cuda()
    L = _bind()
    t0 = time.perf_counter()
    order = int(disc.order)
    nb = order * (order + 1) // 2
    n = disc.nnodes
    # CSR pattern on the device: per row the near patches sorted (the
    # reference's csr_matrix canonical order), nb consecutive columns each
    cuda = "cuda"
    offs = _dev(np.asarray(near.offsets, dtype=np.int64))
    pats = _dev(np.asarray(near.patches, dtype=np.int32))
    npairs = int(offs[-1])
    counts = offs[1:] - offs[:-1]
    tgt = t.repeat_interleave(t.arange(n, device=cuda), counts)
    node_patch = _dev(np.asarray(disc.node_patch, dtype=np.int64))
    key = tgt * int(disc.npatches) + pats.to(t.int64)
    _, order_sorted = t.sort(key, stable=True)
    start = offs[:-1][tgt]
    rank = t.empty_like(order_sorted)
    rank[order_sorted] = t.arange(npairs, device=cuda) - start[order_sorted]
    pair_pos = (start + rank) * nb
    sp = pats[order_sorted].to(t.int64)
    indices = (sp[:, None] * nb + t.arange(nb, device=cuda)[None, :]).reshape(-1).to(t.int32)
    del sp, key, rank
    indptr = offs * nb
    # work order: self pairs (Duffy, ~50x the leaves) first
    is_self = node_patch[tgt] == pats.to(t.int64)
    work = t.cat([t.nonzero(is_self).flatten(), t.nonzero(~is_self).flatten()])
    # geometry in the leaf kernel's layout
    perm = kmajor_permutation(order)
    stacked = np.concatenate([_require(disc, "coeffs_x"), _require(disc, "coeffs_dxdu"),
                              _require(disc, "coeffs_dxdv")], axis=2)
    stacked_km = np.empty_like(stacked)
    stacked_km[:, perm, :] = stacked
    srule, drule = leaf_rules(order)
    over_interp = np.asarray(disc.over_interp if getattr(disc, "over_interp", None)
                             is not None else _require(disc, "over_interp"), dtype=float)
    dev = _dev
    keep = {
        "coeffs": dev(np.ascontiguousarray(stacked_km)),
        "nodes": dev(np.ascontiguousarray(disc.nodes, dtype=float)),
        "normals": dev(np.ascontiguousarray(disc.normals, dtype=float)),
        "node_uv": dev(np.ascontiguousarray(_require(disc, "node_uv"), dtype=float)),
        "node_patch": node_patch,
        "pair_tgt": tgt[work].contiguous(),
        "pair_pat": pats[work].contiguous(),
        "pair_pos": pair_pos[work].contiguous(),
        "srule": dev(np.ascontiguousarray(srule)),
        "drule": dev(np.ascontiguousarray(drule)),
        "knorm": dev(koornwinder_norms_kmajor(order).astype(float)),
        "perm": dev(perm.astype(np.int32)),
        "vinv": dev(np.ascontiguousarray(_vinv(disc))),
        "over_interp": dev(np.ascontiguousarray(over_interp)),
        "over_nodes": dev(np.ascontiguousarray(disc.over_nodes, dtype=float)),
        "over_normals": dev(np.ascontiguousarray(disc.over_normals, dtype=float)),
        "over_weights": dev(np.ascontiguousarray(disc.over_weights, dtype=float)),
    }
    values = {k: t.empty(npairs * nb, dtype=t.float64, device="cuda") for k in kinds}
    d = _Desc()
    d.order = order
    d.nk = len(kinds)
    for i, k in enumerate(kinds):
        d.kinds[i] = KIND_CODE[k]
        d.values[i] = values[k].data_ptr()
    d.eps = float(eps)
    d.coeffs_km = _lib.ptr(keep["coeffs"])
    d.nodes = _lib.ptr(keep["nodes"])
    d.normals = _lib.ptr(keep["normals"])
    d.node_uv = _lib.ptr(keep["node_uv"])
    d.node_patch = _lib.ptr(keep["node_patch"])
    d.pair_tgt = _lib.ptr(keep["pair_tgt"])
    d.pair_pat = _lib.ptr(keep["pair_pat"])
    d.pair_pos = _lib.ptr(keep["pair_pos"])
    d.npairs = npairs
    d.srule = _lib.ptr(keep["srule"])
    d.nqs = srule.shape[0]
    d.drule = _lib.ptr(keep["drule"])
    d.nqd = drule.shape[0]
    d.knorm = _lib.ptr(keep["knorm"])
    d.kmajor_perm = _lib.ptr(keep["perm"])
    d.vinv = _lib.ptr(keep["vinv"])
    d.over_interp = _lib.ptr(keep["over_interp"])
    d.nbo = over_interp.shape[0]
    d.over_nodes = _lib.ptr(keep["over_nodes"])
    d.over_normals = _lib.ptr(keep["over_normals"])
    d.over_weights = _lib.ptr(keep["over_weights"])
    stats = t.zeros(2, dtype=t.int64, device="cuda")
    d.stats = _lib.ptr(stats)
    d.n = n
    if want_pv:
        # principal-value inputs (quadrature.py:436-438, 564-565): mean
        # curvature coefficients per patch (k-major) and the Gauss panel rule
        from scipy.special import roots_legendre
        vinv = np.asarray(_vinv(disc), dtype=float)
        hn = np.asarray(_require(disc, "curvature"), dtype=float).reshape(disc.npatches, nb)
        hco = hn @ vinv.T
        hco_km = np.empty_like(hco)
        hco_km[:, perm] = hco
        gs, gw = roots_legendre(order + 2)
        gauss = np.column_stack([0.5 * (gs + 1.0), 0.5 * gw])
        keep["hcoeff"] = dev(np.ascontiguousarray(hco_km))
        keep["gauss"] = dev(np.ascontiguousarray(gauss))
        d.hcoeff_km = _lib.ptr(keep["hcoeff"])
        d.gauss = _lib.ptr(keep["gauss"])
        d.ng = gauss.shape[0]
    t.cuda.synchronize()
    t1 = time.perf_counter()
    _lib.check(L.lb_corrections_build(ctypes.byref(d), _lib.stream_handle(None)),
               "lb_corrections_build")
    t.cuda.synchronize()
    t2 = time.perf_counter()
    st = stats.cpu().tolist()
    LAST_BUILD.update({"prep_s": t1 - t0, "device_s": t2 - t1, "pairs": npairs,
                       "self_pairs": int(is_self.sum()), "refinements": st[0],
                       "leaves": st[1] + npairs + 2 * int(is_self.sum())})
    cset = CorrectionSet(indptr, indices, values, shape=(n, n))
    return cset, time.perf_counter() - t0


def compute_corrections(disc, near: NearMap, kinds, eps: float):
    """quadrature.py:663-701: (kind -> NearCorrections-like view, t_q)."""
    from .operators import _CorrView
    cset, t_q = build_correction_set(disc, near, kinds, eps)
    return {k: _CorrView(cset, k) for k in cset.values}, t_q
