"""The BASELINE geometries as device-built discretisations.

Each generator samples an analytic chart and its exact first derivatives at
the reference element's interpolation nodes of every parameter triangle
(`shapes.py:27-45` of the reference), turns the samples into per-patch
Koornwinder coefficients with the inverse Vandermonde (`surface.py:310-322`,
host: an (nb x nb) product per patch) and hands them to the device geometry
build (`surface.build_from_coefficients` -> `lb_geom_build`, csrc/geom.cu).
Nothing here reads a file, so the bench and the GPU tests rebuild the configs
on any box.

  icosphere(order)              configs 1-2: the twice 4-way split icosahedron
                                radially projected onto the unit sphere
  build_torus(order, nu, nv, R, r)
                                config 3 (`shapes.py:132-156`): 64 x 32 grid
  wavy_torus(order, nu, nv)     config 4: tube radius 1 + cos(5 phi) sin(3 theta)/4
  sphere_cloud(n, seed)         config 5 point clouds

The parameter grid and its triangle orientation follow `shapes.py:106-129`
(flip=True: X_u x X_v points outward for both torus charts).
"""

from __future__ import annotations

import numpy as np

from .simplex import reference_element

__all__ = ["build_from_samples", "sample_coefficients", "icosphere", "build_torus", "wavy_torus",
           "sphere_cloud", "param_grid_triangles"]


def sample_coefficients(order, x_samples, dxdu_samples, dxdv_samples):
    """Samples (npat, nb, 3) at the interpolation nodes -> chart
    coefficients through the inverse Vandermonde (host, surface.py:317-320)."""
    vinv = reference_element(order).vinv
    return tuple(np.einsum("ij,pjc->pic", vinv, np.asarray(a, dtype=float))
                 for a in (x_samples, dxdu_samples, dxdv_samples))


def build_from_samples(order, x_samples, dxdu_samples, dxdv_samples,
                       node_family="afekete", metadata=None):
    """surface.py:310-322: samples -> coefficients -> device geometry build."""
    from .surface import build_from_coefficients
    return build_from_coefficients(
        order, *sample_coefficients(order, x_samples, dxdu_samples, dxdv_samples),
        node_family=node_family, metadata=metadata)


def _build(order, samples, name, metadata, coefficients_only):
    if coefficients_only:
        return sample_coefficients(order, *samples)
    return _check_outward(build_from_samples(order, *samples, metadata=metadata), name)


def _sample(order, tris, chart):
    """Chart samples on affine parameter triangles tris (npat, 3, 2): the
    point (u, v) of the reference triangle maps to t0 + u (t1 - t0) + v (t2 - t0),
    and the chart derivatives compose with that affine map."""
    uv = reference_element(order).nodes
    tris = np.asarray(tris, dtype=float)
    e1 = tris[:, 1] - tris[:, 0]
    e2 = tris[:, 2] - tris[:, 0]
    p = tris[:, None, 0, :] + uv[None, :, 0, None] * e1[:, None, :] \
        + uv[None, :, 1, None] * e2[:, None, :]
    npat, nb = p.shape[:2]
    x, d1, d2 = chart(p.reshape(-1, 2))
    x, d1, d2 = (a.reshape(npat, nb, 3) for a in (x, d1, d2))
    xu = d1 * e1[:, None, 0, None] + d2 * e1[:, None, 1, None]
    xv = d1 * e2[:, None, 0, None] + d2 * e2[:, None, 1, None]
    return x, xu, xv


def param_grid_triangles(nu: int, nv: int, flip: bool = True):
    """[0, 2pi]^2 cut into nu x nv quads, two triangles each, quads in
    (i, j) row-major order (shapes.py:106-129)."""
    du, dv = 2 * np.pi / nu, 2 * np.pi / nv
    i, j = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    u0, v0 = (i * du).ravel(), (j * dv).ravel()
    a = np.stack([u0, v0], -1)
    b = np.stack([u0 + du, v0], -1)
    c = np.stack([u0 + du, v0 + dv], -1)
    d = np.stack([u0, v0 + dv], -1)
    first = np.stack([a, c, b] if flip else [a, b, c], 1)
    second = np.stack([a, d, c] if flip else [a, c, d], 1)
    return np.stack([first, second], 1).reshape(-1, 3, 2)


def _check_outward(disc, name):
    vol3 = float(np.dot(disc.weights, np.einsum("ik,ik->i", disc.nodes, disc.normals)))
    if vol3 <= 0:
        raise AssertionError(f"{name}: inward orientation (3V = {vol3:.3e})")
    return disc


def build_torus(order: int, nu: int, nv: int, R: float, r: float,
                coefficients_only: bool = False):
    """((R + r cos u) cos v, (R + r cos u) sin v, r sin u) (shapes.py:132-156)."""
    if R <= r or r <= 0:
        raise ValueError("torus requires R > r > 0")
    if nu < 4 or nv < 4:
        raise ValueError("nu, nv must be >= 4")

    def chart(p):
        u, v = p[:, 0], p[:, 1]
        cu, su, cv, sv = np.cos(u), np.sin(u), np.cos(v), np.sin(v)
        ring = R + r * cu
        x = np.stack([ring * cv, ring * sv, r * su], -1)
        xu = np.stack([-r * su * cv, -r * su * sv, r * cu], -1)
        xv = np.stack([-ring * sv, ring * cv, np.zeros_like(u)], -1)
        return x, xu, xv
    return _build(order, _sample(order, param_grid_triangles(nu, nv), chart), "torus",
                  {"geometry": "torus", "R": R, "r": r, "nu": nu, "nv": nv},
                  coefficients_only)


def wavy_torus(order: int = 9, nu: int = 82, nv: int = 163,
               coefficients_only: bool = False):
    """BASELINE config 4: tube radius rho(theta, phi) = 1 + cos(5 phi) sin(3 theta)/4
    around the R = 2 circle; theta poloidal on the u axis, phi toroidal on the
    v axis (SURVEY §8(d) config 4 chart, validated there against the
    reference's outward check)."""
    def chart(p):
        th, ph = p[:, 0], p[:, 1]
        rho = 1.0 + 0.25 * np.cos(5 * ph) * np.sin(3 * th)
        rho_t = 0.75 * np.cos(5 * ph) * np.cos(3 * th)
        rho_p = -1.25 * np.sin(5 * ph) * np.sin(3 * th)
        zero = np.zeros_like(ph)
        er = np.stack([np.cos(ph), np.sin(ph), zero], -1)
        ep = np.stack([-np.sin(ph), np.cos(ph), zero], -1)
        ez = np.array([0.0, 0.0, 1.0])
        ring = 2.0 + rho * np.cos(th)
        x = ring[:, None] * er + (rho * np.sin(th))[:, None] * ez
        xt = (rho_t * np.cos(th) - rho * np.sin(th))[:, None] * er \
            + (rho_t * np.sin(th) + rho * np.cos(th))[:, None] * ez
        xp = (rho_p * np.cos(th))[:, None] * er + ring[:, None] * ep \
            + (rho_p * np.sin(th))[:, None] * ez
        return x, xt, xp
    return _build(order, _sample(order, param_grid_triangles(nu, nv), chart), "wavy-torus",
                  {"geometry": "wavy-torus", "nu": nu, "nv": nv}, coefficients_only)


def _icosahedron():
    """12 unit vertices (cyclic permutations of (0, +-1, +-golden)) and the 20
    faces, wound so the face normal points away from the origin."""
    g = (1.0 + 5 ** 0.5) / 2.0
    v = np.array([p for a in (-1.0, 1.0) for b in (-g, g)
                  for p in ((0.0, a, b), (a, b, 0.0), (b, 0.0, a))])
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    d = np.linalg.norm(v[:, None] - v[None], axis=-1)
    edge = d[d > 1e-9].min()
    adj = np.abs(d - edge) < 1e-9
    faces = []
    for i in range(12):
        for j in range(i + 1, 12):
            for k in range(j + 1, 12):
                if adj[i, j] and adj[i, k] and adj[j, k]:
                    nrm = np.cross(v[j] - v[i], v[k] - v[i])
                    faces.append([i, j, k] if np.dot(nrm, v[i] + v[j] + v[k]) > 0
                                 else [i, k, j])
    return v, np.array(faces)


def _split4(t):
    """The four uniform children of each triangle t (..., 3, 3), in the
    child order of simplex.py:280-290."""
    m01 = 0.5 * (t[:, 0] + t[:, 1])
    m12 = 0.5 * (t[:, 1] + t[:, 2])
    m20 = 0.5 * (t[:, 2] + t[:, 0])
    kids = np.stack([np.stack([t[:, 0], m01, m20], 1), np.stack([m01, t[:, 1], m12], 1),
                     np.stack([m20, m12, t[:, 2]], 1), np.stack([m01, m12, m20], 1)], 1)
    return kids.reshape(-1, 3, 3)


def icosphere(order: int, nsplit: int = 2, coefficients_only: bool = False):
    """BASELINE configs 1-2: 20 * 4^nsplit flat triangles (320 at nsplit = 2)
    projected radially onto the unit sphere, X = c / |c| with
    dX = (I - X X^T) dc / |c| (the projection math of shapes.py:85-93)."""
    v, f = _icosahedron()
    tris = v[f]
    for _ in range(nsplit):
        tris = _split4(tris)
    uv = reference_element(order).nodes
    e1 = tris[:, 1] - tris[:, 0]
    e2 = tris[:, 2] - tris[:, 0]
    c = tris[:, None, 0] + uv[None, :, 0, None] * e1[:, None] + uv[None, :, 1, None] * e2[:, None]
    r = np.linalg.norm(c, axis=-1, keepdims=True)
    x = c / r

    def proj(dc):
        return (dc - x * np.einsum("pik,pik->pi", x, dc)[..., None]) / r
    xu = proj(np.broadcast_to(e1[:, None], c.shape))
    xv = proj(np.broadcast_to(e2[:, None], c.shape))
    return _build(order, (x, xu, xv), "icosphere",
                  {"geometry": "icosphere", "nsplit": nsplit}, coefficients_only)


def sphere_cloud(n: int, seed: int = 105):
    """BASELINE config 5: default_rng(seed) standard normals normalised onto
    the unit sphere (seed 100 + config)."""
    x = np.random.default_rng(seed).standard_normal((n, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x
