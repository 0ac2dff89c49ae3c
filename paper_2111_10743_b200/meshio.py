"""The lbmesh text format (meshio.py:17-50): a versioned header
`lbmesh 1 npat P order p family F` followed, per patch, by the Koornwinder
coefficient blocks of X, X_u and X_v (nb rows of three `%.17g` numbers each).

`write_mesh` emits byte-identical files to the reference's writer for the
same coefficients; `read_mesh` parses them with the reference's header
checks and error messages and rebuilds the discretization on the device
(`surface.build_from_coefficients`).  VTK output (meshio.py:53-120) is a
visualisation aid outside the solve path.
"""

from __future__ import annotations

import numpy as np

from .simplex import basis_size
from .surface import build_from_coefficients

__all__ = ["MAGIC", "VERSION", "write_mesh", "read_mesh", "read_coefficients"]

MAGIC = "lbmesh"
VERSION = 1


def write_mesh(path, disc):
    """Header + (X, X_u, X_v) blocks per patch (meshio.py:21-32)."""
    cx = np.asarray(disc.coeffs_x, dtype=float)
    cu = np.asarray(disc.coeffs_dxdu, dtype=float)
    cv = np.asarray(disc.coeffs_dxdv, dtype=float)
    npat = cx.shape[0]
    family = getattr(disc, "node_family", None) or \
        getattr(disc, "metadata", {}).get("node_family", "afekete")
    # one (npat, 3, nb, 3) block array written row by row, %.17g round-trips
    blocks = np.stack([cx, cu, cv], axis=1).reshape(-1, 3)
    with open(path, "w") as fh:
        fh.write(f"{MAGIC} {VERSION} npat {npat} order {disc.order} "
                 f"family {family}\n")
        fh.writelines("%.17g %.17g %.17g\n" % (a, b, c) for a, b, c in blocks)


def read_coefficients(path):
    """Parse an lbmesh file -> (order, family, coeffs (npat, 3, nb, 3)),
    raising the reference's ValueErrors for a bad magic, version or header
    (meshio.py:35-48)."""
    with open(path) as fh:
        header = fh.readline().split()
        if len(header) != 8 or header[0] != MAGIC:
            raise ValueError(f"{path}: not an lbmesh file")
        if int(header[1]) != VERSION:
            raise ValueError(f"{path}: unsupported lbmesh version {header[1]}")
        if header[2] != "npat" or header[4] != "order" or header[6] != "family":
            raise ValueError(f"{path}: malformed lbmesh header")
        npat, order, family = int(header[3]), int(header[5]), header[7]
        nb = basis_size(order)
        data = np.loadtxt(fh).reshape(npat, 3, nb, 3)
    return order, family, data


def read_mesh(path):
    """Read an lbmesh file and rebuild the full discretization on the B200
    (meshio.py:35-50)."""
    order, family, data = read_coefficients(path)
    return build_from_coefficients(order, data[:, 0], data[:, 1], data[:, 2],
                                   node_family=family,
                                   metadata={"source": str(path)})
