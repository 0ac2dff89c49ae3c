"""Config 3's post-processing on the host (paper_2111_10743_b200/hodge.py)
against the reference's own hodge_decompose output on the reduced 12 x 6
torus (tests/golden/hodge_torus_o7.npz, scripts/make_golden_r2.py
hodge_small): the surface calculus (surface.py:335-367) reproduces the
reference's grad alpha, n x grad beta and H from the reference's alpha and
beta, and the BASELINE Gaussian field is the reference's field.  No device."""

import numpy as np

from conftest import golden


def _geom(g):
    from paper_2111_10743_b200.operators import Geometry
    geo = Geometry.from_arrays(g)
    geo.sqrt_det_g = g["sqrt_det_g"]
    return geo


def test_surface_calculus_matches_reference():
    from paper_2111_10743_b200.hodge import surface_gradient
    g = golden("hodge_torus_o7.npz")
    geo = _geom(g)
    ga = surface_gradient(geo, g["alpha"])
    rb = np.cross(geo.normals, surface_gradient(geo, g["beta"]))
    assert np.abs(ga - g["grad_alpha"]).max() <= 1e-13 * np.abs(g["grad_alpha"]).max()
    assert np.abs(rb - g["rot_beta"]).max() <= 1e-13 * np.abs(g["rot_beta"]).max()
    h = g["field"] - ga - rb
    h -= np.einsum("ik,ik->i", h, geo.normals)[:, None] * geo.normals
    assert np.abs(h - g["harmonic"]).max() <= 1e-12 * np.abs(g["field"]).max()


def test_divergence_norms_match_reference():
    from paper_2111_10743_b200.hodge import surface_divergence
    g = golden("hodge_torus_o7.npz")
    geo = _geom(g)
    h = g["field"] - g["grad_alpha"] - g["rot_beta"]
    w = geo.weights
    d = surface_divergence(geo, h)
    dn = surface_divergence(geo, np.cross(geo.normals, h))
    assert abs(np.sqrt(np.dot(w, d * d)) - float(g["div_h_norm"])) <= 1e-10 * float(g["div_h_norm"])
    assert abs(np.sqrt(np.dot(w, dn * dn)) - float(g["div_nxh_norm"])) <= 1e-10 * float(g["div_nxh_norm"])


def test_gaussian_field_is_the_reference_field():
    from paper_2111_10743_b200.hodge import gaussian_field
    g = golden("hodge_torus_o7.npz")
    f = gaussian_field(_geom(g))
    assert np.abs(f.values - g["field"]).max() <= 1e-14 * np.abs(g["field"]).max()
