"""Golden fixtures for the reference-element tables and the lbmesh format,
made by running the REFERENCE package (lapbel) in this container.  Test
infrastructure only: nothing in the product imports this.

    python scripts/make_golden_mesh.py

writes
  tests/golden/refelem_sha256.json  SHA-256 of every ReferenceElement field
                                    (simplex.py:359-397), orders 2-10
  tests/golden/twisted_torus_o5.lbmesh  the reference's write_mesh output
                                    (meshio.py:21-32) for
                                    build_twisted_torus(5, 6, 4)
  tests/golden/mesh_twisted_torus_o5.npz  the reference's read_mesh of that
                                    file (meshio.py:35-50 ->
                                    build_from_coefficients): every array
                                    field of the SurfaceDiscretization
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_lapbel")
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from lapbel import meshio, shapes  # noqa: E402
from lapbel.simplex import reference_element  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")

FIELDS = ["nodes", "node_patch", "node_uv", "tangents_u", "tangents_v",
          "normals", "metric", "inv_metric", "sqrt_det_g", "curvature",
          "weights", "over_nodes", "over_patch", "over_uv", "over_normals",
          "over_weights", "coeffs_x", "coeffs_dxdu", "coeffs_dxdv"]


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(str(a.dtype).encode() + str(a.shape).encode()
                          + a.tobytes()).hexdigest()


def main():
    digests = {}
    for order in range(2, 11):
        ref = reference_element(order)
        digests[str(order)] = {
            f: (sha(getattr(ref, f)) if isinstance(getattr(ref, f), np.ndarray)
                else int(getattr(ref, f)))
            for f in ref.__dataclass_fields__}
    with open(os.path.join(GOLD, "refelem_sha256.json"), "w") as fh:
        json.dump({"generator": "lapbel.simplex.reference_element",
                   "orders": digests}, fh, indent=1)

    disc = shapes.build_twisted_torus(5, 6, 4)
    path = os.path.join(GOLD, "twisted_torus_o5.lbmesh")
    meshio.write_mesh(path, disc)
    back = meshio.read_mesh(path)
    arrs = {f: np.asarray(getattr(back, f)) for f in FIELDS}
    arrs["order"] = np.int64(back.order)
    arrs["family"] = np.array(back.node_family)
    np.savez_compressed(os.path.join(GOLD, "mesh_twisted_torus_o5.npz"), **arrs)
    print("npatches", back.npatches, "N", back.nnodes)


if __name__ == "__main__":
    main()
