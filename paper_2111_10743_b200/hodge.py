"""BASELINE config 3's workload: the Hodge decomposition of a tangential field
(`hodge.py:126-161` of the reference) -- two Laplace-Beltrami solves on ONE
device operator set, with the reference's surface calculus around them.

  F = grad(alpha) + n x grad(beta) + H,
  lap alpha = div F,   lap beta = -div (n x F)

The two solves are this package's device GMRES + operator apply (the hot
path).  The surface calculus (`surface.py:335-367`: per-patch spectral
differentiation with the reference element's dmat_u / dmat_v, the inverse
metric and sqrt(det g)) is the reference's host post-processing, restated
here on the host in numpy: it is O(N nb) work outside the apply, run twice
per decomposition.

`gaussian_field` is config 3's input: the tangential projection of a sum of
16 seeded Gaussians (width 0.5) with N(0,1) vector amplitudes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .operators import DensityVector
from .simplex import reference_element
from .solver import SolveConfig, solve_laplace_beltrami

__all__ = ["TangentialField", "HodgeResult", "hodge_decompose", "surface_gradient",
           "surface_divergence", "gaussian_field"]


def _sqrt_det_g(disc):
    sg = getattr(disc, "sqrt_det_g", None)
    if sg is not None:
        return np.asarray(sg)
    return np.linalg.norm(np.cross(disc.tangents_u, disc.tangents_v), axis=1)


def _patch_derivatives(disc, f):
    """d/du, d/dv of a node-sampled scalar per patch (surface.py:165-172)."""
    ref = reference_element(disc.order)
    fp = np.asarray(f, dtype=float).reshape(-1, ref.dmat_u.shape[0])
    return (fp @ ref.dmat_u.T).ravel(), (fp @ ref.dmat_v.T).ravel()


def surface_gradient(disc, f):
    """Tangential gradient (N, 3) of a node-sampled scalar (surface.py:335-341):
    g^{ij} d_j f X_i."""
    du, dv = _patch_derivatives(disc, f)
    gi = disc.inv_metric
    a = gi[:, 0, 0] * du + gi[:, 0, 1] * dv
    b = gi[:, 1, 0] * du + gi[:, 1, 1] * dv
    return a[:, None] * disc.tangents_u + b[:, None] * disc.tangents_v


def surface_divergence(disc, field_xyz):
    """Surface divergence of a node-sampled field (surface.py:344-367): the
    normal part projected out, chart components F^i = g^{ij} (F . X_j), then
    (d_1 (sg F^1) + d_2 (sg F^2)) / sg."""
    F = np.asarray(field_xyz, dtype=float)
    n = disc.normals
    Ft = F - np.einsum("ik,ik->i", F, n)[:, None] * n
    fu = np.einsum("ik,ik->i", Ft, disc.tangents_u)
    fv = np.einsum("ik,ik->i", Ft, disc.tangents_v)
    gi = disc.inv_metric
    f1 = gi[:, 0, 0] * fu + gi[:, 0, 1] * fv
    f2 = gi[:, 1, 0] * fu + gi[:, 1, 1] * fv
    sg = _sqrt_det_g(disc)
    d1, _ = _patch_derivatives(disc, sg * f1)
    _, d2 = _patch_derivatives(disc, sg * f2)
    return (d1 + d2) / sg


@dataclass
class TangentialField:
    """A tangential field sampled at the nodes (N, 3) (hodge.py:40-66)."""

    values: np.ndarray
    tangency_residual: float = 0.0

    @classmethod
    def project(cls, disc, vfield):
        """V - (V . n) n (hodge.py:47-54)."""
        v = np.asarray(vfield, dtype=float)
        f = v - np.einsum("ik,ik->i", v, disc.normals)[:, None] * disc.normals
        resid = float(np.abs(np.einsum("ik,ik->i", f, disc.normals)).max())
        return cls(values=f, tangency_residual=resid / (np.abs(f).max() + 1e-300))

    def rotate(self, disc):
        return TangentialField(np.cross(disc.normals, self.values), self.tangency_residual)


@dataclass
class HodgeResult:
    """hodge.py:69-81."""

    alpha: DensityVector
    beta: DensityVector
    grad_alpha: TangentialField
    rot_beta: TangentialField
    harmonic: TangentialField
    div_h_norm: float
    div_nxh_norm: float
    n_iter: tuple
    converged: bool
    t_s: float
    reports: tuple


def hodge_decompose(opset, field: TangentialField, cfg: SolveConfig | None = None):
    """hodge.py:126-161: two solves on the shared (device) operator set."""
    disc = opset.disc
    f = field.values
    rhs_alpha = surface_divergence(disc, f)
    rhs_beta = -surface_divergence(disc, np.cross(disc.normals, f))
    rep_a = solve_laplace_beltrami(opset, rhs_alpha, cfg)
    rep_b = solve_laplace_beltrami(opset, rhs_beta, cfg)
    ua, ub = np.asarray(rep_a.u.values), np.asarray(rep_b.u.values)
    grad_alpha = surface_gradient(disc, ua)
    rot_beta = np.cross(disc.normals, surface_gradient(disc, ub))
    h = f - grad_alpha - rot_beta
    w = disc.weights

    def l2(v):
        return float(np.sqrt(max(float(np.dot(w, v * v)), 0.0)))
    return HodgeResult(
        alpha=DensityVector(ua, "solution_u"), beta=DensityVector(ub, "solution_u"),
        grad_alpha=TangentialField(grad_alpha), rot_beta=TangentialField(rot_beta),
        harmonic=TangentialField.project(disc, h),
        div_h_norm=l2(surface_divergence(disc, h)),
        div_nxh_norm=l2(surface_divergence(disc, np.cross(disc.normals, h))),
        n_iter=(rep_a.n_iter, rep_b.n_iter), converged=rep_a.converged and rep_b.converged,
        t_s=rep_a.t_s + rep_b.t_s, reports=(rep_a, rep_b))


def gaussian_field(disc, seed_amp: int = 3, seed_centres: int = 103, k: int = 16,
                   width: float = 0.5) -> TangentialField:
    """BASELINE config 3's field: the tangential projection of
    sum_k a_k exp(-|x - c_k|^2 / (2 width^2)) with a_k ~ N(0,1)^3 from
    default_rng(seed_amp) and centres c_k = nodes picked by
    default_rng(seed_centres) (seed 100 + config)."""
    nodes = disc.nodes
    cen = nodes[np.random.default_rng(seed_centres).choice(len(nodes), k, replace=False)]
    amp = np.random.default_rng(seed_amp).standard_normal((k, 3))
    d2 = ((nodes[:, None, :] - cen[None, :, :]) ** 2).sum(-1)
    return TangentialField.project(disc, np.exp(-d2 / (2 * width ** 2)) @ amp)
