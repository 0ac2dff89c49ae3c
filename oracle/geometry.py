"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Host numpy restatement of the geometry evaluation of
build_from_coefficients (surface.py:176-307) -- nodes, normals, mean
curvature, smooth weights and the oversampled set -- so the CPU reference
arm of bench.py can build a BASELINE geometry without the device library.
The reference-element tables come from the host module
paper_2111_10743_b200.simplex (pure numpy, SHA-256-identical to the
reference's, tests/test_mesh_cpu.py); nothing here touches CUDA.
"""

from __future__ import annotations

import numpy as np


def evaluate(order, cx, cu, cv):
    """Chart coefficients (npat, nb, 3) -> the arrays the apply consumes."""
    from paper_2111_10743_b200.simplex import CHILD_TRIANGLES, interpolation_nodes, \
        koornwinder, reference_element
    ref = reference_element(order)
    npat, nb, _ = cx.shape

    def at(psi, c):                       # (q, nb) x (npat, nb, 3) -> (npat, q, 3)
        return np.einsum("qj,pjc->pqc", psi, c)

    x, xu, xv = at(ref.vand, cx), at(ref.vand, cu), at(ref.vand, cv)
    cr = np.cross(xu, xv)
    jac = np.linalg.norm(cr, axis=-1)
    nrm = cr / jac[..., None]
    g11 = (xu * xu).sum(-1)
    g12 = (xu * xv).sum(-1)
    g22 = (xv * xv).sum(-1)
    det = g11 * g22 - g12 * g12
    # H = -(1/2) g^{ij} n . X_ij with the second derivatives from the
    # spectral derivative matrices applied to the stored tangents
    xuu = at(ref.dmat_u, xu)
    xvv = at(ref.dmat_v, xv)
    xuv = 0.5 * (at(ref.dmat_v, xu) + at(ref.dmat_u, xv))
    b11, b12, b22 = ((nrm * a).sum(-1) for a in (xuu, xuv, xvv))
    curv = -0.5 * (g22 * b11 - 2.0 * g12 * b12 + g11 * b22) / det
    rp = ref.rule_pts
    psi_rule = koornwinder(order, rp[:, 0], rp[:, 1])
    jr = np.linalg.norm(np.cross(at(psi_rule, cu), at(psi_rule, cv)), axis=-1)
    weights = np.einsum("qi,pq->pi", ref.weight_interp, jr * ref.rule_wts)
    psi_o = koornwinder(order, ref.over_pts[:, 0], ref.over_pts[:, 1])
    ox = at(psi_o, cx)
    ocr = np.cross(at(psi_o, cu), at(psi_o, cv))
    onrm = ocr / np.linalg.norm(ocr, axis=-1)[..., None]
    no4 = ref.over_pts.shape[0] // 4
    on = interpolation_nodes(ref.over_order)
    w_o = koornwinder(ref.over_order, rp[:, 0], rp[:, 1]) @ np.linalg.inv(
        koornwinder(ref.over_order, on[:, 0], on[:, 1]))
    ow = np.empty((npat, 4 * no4))
    for k, tri in enumerate(CHILD_TRIANGLES):
        q = tri[0] + np.outer(rp[:, 0], tri[1] - tri[0]) + np.outer(rp[:, 1], tri[2] - tri[0])
        psi_q = koornwinder(order, q[:, 0], q[:, 1])
        jq = np.linalg.norm(np.cross(at(psi_q, cu), at(psi_q, cv)), axis=-1)
        ow[:, k * no4:(k + 1) * no4] = np.einsum("qi,pq->pi", w_o, 0.25 * jq * ref.rule_wts)
    return {"order": order, "nb": nb, "npatches": npat,
            "nodes": x.reshape(-1, 3), "normals": nrm.reshape(-1, 3),
            "curvature": curv.ravel(), "weights": weights.ravel(),
            "over_nodes": ox.reshape(-1, 3), "over_normals": onrm.reshape(-1, 3),
            "over_weights": ow.ravel(), "over_interp": ref.over_interp,
            "node_patch": np.repeat(np.arange(npat), nb)}


def near_patches(nodes, npatches, nb, over_nodes, targets, eta=2.0):
    """build_near_map (quadrature.py:76-104) for a subset of targets, by
    brute force over the patch bounding spheres (centre = mean of the
    patch's nodes and oversampled nodes, radius = max distance,
    surface.py:146-153): own patch first, then ascending patch index."""
    pos = nodes.reshape(npatches, nb, 3)
    over = over_nodes.reshape(npatches, -1, 3)
    allp = np.concatenate([pos, over], axis=1)
    cen = allp.mean(axis=1)
    rad = np.sqrt(((allp - cen[:, None, :]) ** 2).sum(-1)).max(axis=1)
    out = []
    for t in targets:
        d = np.sqrt(((cen - nodes[t]) ** 2).sum(-1))
        own = t // nb
        hit = np.nonzero(d <= (1.0 + eta) * rad)[0]
        out.append(np.concatenate([[own], hit[hit != own]]).astype(np.int64))
    return out
