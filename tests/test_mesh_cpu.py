"""Reference-element tables and the lbmesh format on the CPU (no device):
the restated simplex.py tables are BIT-IDENTICAL to the reference's
(SHA-256 of every ReferenceElement field, orders 2-10, written by
scripts/make_golden_mesh.py from lapbel), the writer reproduces the
reference's file byte for byte, and the reader raises the reference's
errors on bad headers (meshio.py:38-45)."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLD, golden

MESH = os.path.join(GOLD, "twisted_torus_o5.lbmesh")


def _sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(str(a.dtype).encode() + str(a.shape).encode()
                          + a.tobytes()).hexdigest()


@pytest.mark.parametrize("order", list(range(2, 11)))
def test_reference_element_bit_identical(order):
    from paper_2111_10743_b200.simplex import reference_element
    with open(os.path.join(GOLD, "refelem_sha256.json")) as fh:
        want = json.load(fh)["orders"][str(order)]
    ref = reference_element(order)
    for field, digest in want.items():
        got = getattr(ref, field)
        if isinstance(got, np.ndarray):
            assert _sha(got) == digest, field
        else:
            assert got == digest, field


def test_koornwinder_orthonormal():
    # orthonormal on T0 with respect to area (simplex.py:68-75): the
    # order-(p+1) collapsed rule integrates degree <= 2p+1 exactly
    from paper_2111_10743_b200.simplex import koornwinder, triangle_rule
    pts, w = triangle_rule(8)
    psi = koornwinder(7, pts[:, 0], pts[:, 1])
    np.testing.assert_allclose((psi * w[:, None]).T @ psi, np.eye(28),
                               atol=1e-13)
    assert abs(w.sum() - 0.5) < 1e-15


def test_read_coefficients_matches_reference_reader():
    from paper_2111_10743_b200.meshio import read_coefficients
    order, family, data = read_coefficients(MESH)
    g = golden("mesh_twisted_torus_o5.npz")
    assert order == int(g["order"]) and family == str(g["family"])
    np.testing.assert_array_equal(data[:, 0], g["coeffs_x"])
    np.testing.assert_array_equal(data[:, 1], g["coeffs_dxdu"])
    np.testing.assert_array_equal(data[:, 2], g["coeffs_dxdv"])


def test_write_mesh_byte_identical(tmp_path):
    from paper_2111_10743_b200.meshio import read_coefficients, write_mesh

    class Disc:  # the fields write_mesh reads (meshio.py:21-32)
        pass

    order, family, data = read_coefficients(MESH)
    d = Disc()
    d.order, d.node_family = order, family
    d.coeffs_x, d.coeffs_dxdu, d.coeffs_dxdv = data[:, 0], data[:, 1], data[:, 2]
    out = tmp_path / "o.lbmesh"
    write_mesh(out, d)
    assert out.read_bytes() == open(MESH, "rb").read()


@pytest.mark.parametrize("header,msg", [
    ("lbmsh 1 npat 1 order 2 family afekete", "not an lbmesh file"),
    ("lbmesh 1 npat 1 order 2", "not an lbmesh file"),
    ("lbmesh 2 npat 1 order 2 family afekete", "unsupported lbmesh version 2"),
    ("lbmesh 1 npatch 1 order 2 family afekete", "malformed lbmesh header"),
])
def test_read_mesh_header_errors(tmp_path, header, msg):
    from paper_2111_10743_b200.meshio import read_mesh
    p = tmp_path / "bad.lbmesh"
    p.write_text(header + "\n" + "0 0 0\n" * 9)
    with pytest.raises(ValueError, match=msg):
        read_mesh(p)


def test_build_rejects_order_mismatch():
    # surface.py:190-191, raised before any device work
    from paper_2111_10743_b200.surface import build_from_coefficients
    c = np.zeros((2, 6, 3))
    with pytest.raises(ValueError, match="do not match the stated order"):
        build_from_coefficients(4, c, c, c)
