"""`build_from_coefficients` (surface.py:176-307): a surface discretization
assembled from per-patch chart expansions -- the constructor behind the
lbmesh reader (`meshio.read_mesh`).

The reference-element tables are the host precompute of `simplex.py`
(bit-identical to the reference's); every per-patch quantity (nodes,
tangents, normals, metric, mean curvature, smooth weights, the oversampled
set) is evaluated on the B200 by `lb_geom_build` (csrc/geom.cu), one CTA per
patch.  The result is a `Geometry` the operator set, near map and correction
build consume directly.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .operators import Geometry
from .simplex import (CHILD_TRIANGLES, basis_size, interpolation_nodes,
                      koornwinder, reference_element)

__all__ = ["MIN_JACOBIAN", "DegeneratePatchError", "SurfaceDiscretization",
           "build_from_coefficients"]

MIN_JACOBIAN = 1e-14  # surface.py:39


class DegeneratePatchError(RuntimeError):
    """A patch chart has |X_u x X_v| below the degeneracy floor (surface.py:42-43)."""


@dataclass
class SurfaceDiscretization(Geometry):
    """Geometry plus the remaining SurfaceDiscretization fields
    (surface.py:77-106) the reader returns."""

    metric: np.ndarray | None = None
    sqrt_det_g: np.ndarray | None = None
    over_patch: np.ndarray | None = None
    over_uv: np.ndarray | None = None
    node_family: str = "afekete"


class _GeomDesc(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int), ("nb", ctypes.c_int),
                ("nq", ctypes.c_int), ("no", ctypes.c_int),
                ("npatches", ctypes.c_int64)] + [
        (name, ctypes.c_void_p) for name in (
            "coeffs_x", "coeffs_dxdu", "coeffs_dxdv", "vand", "dmat_u",
            "dmat_v", "psi_rule", "rule_wts", "weight_interp", "psi_over",
            "psi_child", "w_interp_o", "nodes", "tangents_u", "tangents_v",
            "normals", "metric", "inv_metric", "sqrt_det_g", "curvature",
            "weights", "over_nodes", "over_normals", "over_weights", "stats")]


@lru_cache(maxsize=16)
def geometry_tables(order: int):
    """Host tables for lb_geom_build: the reference element's operators plus
    the basis on the smooth rule, at the oversampled points, on the rule
    mapped into each child triangle, and the order-`over_order`
    rule-to-node pull-back (surface.py:250-283)."""
    ref = reference_element(order)
    rp = ref.rule_pts
    psi_rule = koornwinder(order, rp[:, 0], rp[:, 1])
    psi_over = koornwinder(order, ref.over_pts[:, 0], ref.over_pts[:, 1])
    onodes = interpolation_nodes(ref.over_order)
    over_vinv = np.linalg.inv(koornwinder(ref.over_order, onodes[:, 0],
                                          onodes[:, 1]))
    w_interp_o = koornwinder(ref.over_order, rp[:, 0], rp[:, 1]) @ over_vinv
    child = []
    for tri in CHILD_TRIANGLES:
        quv = tri[0] + np.outer(rp[:, 0], tri[1] - tri[0]) \
            + np.outer(rp[:, 1], tri[2] - tri[0])
        child.append(koornwinder(order, quv[:, 0], quv[:, 1]))
    return {"vand": ref.vand, "dmat_u": ref.dmat_u, "dmat_v": ref.dmat_v,
            "psi_rule": psi_rule, "rule_wts": ref.rule_wts,
            "weight_interp": ref.weight_interp, "psi_over": psi_over,
            "psi_child": np.stack(child), "w_interp_o": w_interp_o}


def build_from_coefficients(order, coeffs_x, coeffs_dxdu, coeffs_dxdv,
                            node_family="afekete", metadata=None,
                            consistency_tol=0.2) -> SurfaceDiscretization:
    """Same arguments, checks and error types as surface.py:176-307:
    ValueError when nb does not match the order or when the stored
    derivative expansions disagree with the differentiated chart beyond
    max(consistency_tol, 60 * tail * order); DegeneratePatchError when
    |X_u x X_v| < 1e-14 at a node or an oversampled node."""
    cx = np.ascontiguousarray(coeffs_x, dtype=float)
    cu = np.ascontiguousarray(coeffs_dxdu, dtype=float)
    cv = np.ascontiguousarray(coeffs_dxdv, dtype=float)
    if cx.ndim != 3 or cx.shape[2] != 3 or cu.shape != cx.shape \
            or cv.shape != cx.shape:
        raise ValueError("coefficient arrays must be (npatches, nb, 3) alike")
    npat, nb, _ = cx.shape
    if nb != basis_size(order):
        raise ValueError("coefficient arrays do not match the stated order")
    _lib.require_cuda()
    ref = reference_element(order)
    tabs = {k: _lib.to_device(v) for k, v in geometry_tables(order).items()}
    nq = ref.rule_pts.shape[0]
    no = ref.over_pts.shape[0]
    n, nov = npat * nb, npat * no
    out = {
        "nodes": (n, 3), "tangents_u": (n, 3), "tangents_v": (n, 3),
        "normals": (n, 3), "metric": (n, 2, 2), "inv_metric": (n, 2, 2),
        "sqrt_det_g": (n,), "curvature": (n,), "weights": (n,),
        "over_nodes": (nov, 3), "over_normals": (nov, 3),
        "over_weights": (nov,), "stats": (6,)}
    dev = {k: _lib.empty(s) for k, s in out.items()}
    dc = {"coeffs_x": _lib.to_device(cx), "coeffs_dxdu": _lib.to_device(cu),
          "coeffs_dxdv": _lib.to_device(cv)}
    d = _GeomDesc(order=order, nb=nb, nq=nq, no=no, npatches=npat)
    for k, v in {**dc, **tabs, **dev}.items():
        setattr(d, k, v.data_ptr())
    _lib.call("lb_geom_build", ctypes.byref(d), _lib.stream_handle())
    host = {k: v.cpu().numpy() for k, v in dev.items()}
    mis, scale, jmin, ojmin, top2, all2 = host.pop("stats")
    # surface.py:199-215 (the stats are exact maxima/minima; the norms are
    # sums whose order differs from numpy's, irrelevant at this tolerance)
    mismatch = mis / (scale + 1e-300)
    tail = np.sqrt(top2) / (np.sqrt(all2) + 1e-300)
    tol = max(consistency_tol, 60.0 * tail * order)
    if mismatch > tol:
        raise ValueError(
            f"stored chart derivatives disagree with the differentiated "
            f"chart expansion (relative mismatch {mismatch:.2e}, allowed "
            f"{tol:.2e}); check coefficient wiring")
    if npat and jmin < MIN_JACOBIAN:
        raise DegeneratePatchError(
            f"degenerate patch: min |X_u x X_v| = {jmin:.3e}")
    if npat and ojmin < MIN_JACOBIAN:
        raise DegeneratePatchError("degenerate patch at oversampled nodes")
    md = dict(metadata or {})
    md.setdefault("node_family", node_family)
    md.setdefault("oversampling", 4)
    return SurfaceDiscretization(
        order=order, over_interp=ref.over_interp, vinv=ref.vinv,
        coeffs_x=cx, coeffs_dxdu=cu, coeffs_dxdv=cv,
        node_patch=np.repeat(np.arange(npat), nb),
        node_uv=np.tile(ref.nodes, (npat, 1)),
        over_patch=np.repeat(np.arange(npat), no),
        over_uv=np.tile(ref.over_pts, (npat, 1)),
        node_family=node_family, metadata=md, **host)
