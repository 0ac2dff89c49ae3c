"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The A3 operator apply (operators.py:229-266, use_fmm=False: exact far sums)
evaluated at a SUBSET of target rows -- the row-sampled form of the oracle
used (a) by tests/ to check the device apply of the BASELINE-scale configs
at sampled rows, and (b) by bench.py's CPU reference arm to time a bounded
sample of the config-3 apply on the host cores (scaled by N / rows).

Both far calls run over ALL oversampled sources with the targets restricted
to `rows` (oracle.p2p in C, OpenMP); the corrections are CSR rows of the
sampled targets only (columns over all N nodes).  Pass 2's densities
mu1 = S' tau and mu2 = S tau are needed at EVERY node (they are the second
call's sources): the caller passes them (`mu`), e.g. the device's own pass-1
vectors in a parity test; timing runs pass substitutes of the same size
(the cost does not depend on the values).
"""

from __future__ import annotations

import numpy as np

from .core import FOUR_PI, csr_matvec, p2p


class SampledA3:
    def __init__(self, geo, rows, corr, nthreads=0):
        """geo: dict of the geometry arrays (nodes, normals, weights,
        curvature, over_nodes, over_normals, over_weights, over_interp);
        rows: sampled target indices; corr: dict with 'indptr' (len(rows)+1),
        'indices' and per-kind values 's', 'sprime', 'spp_plus_dprime' for
        those rows."""
        self.rows = np.asarray(rows, dtype=np.int64)
        self.nodes = np.ascontiguousarray(geo["nodes"][self.rows])
        self.normals = np.ascontiguousarray(geo["normals"][self.rows])
        self.curv = np.asarray(geo["curvature"])[self.rows]
        self.weights = np.asarray(geo["weights"])
        self.over = np.ascontiguousarray(geo["over_nodes"])
        self.overn = np.ascontiguousarray(geo["over_normals"])
        self.wover = np.asarray(geo["over_weights"])
        self.oi = np.asarray(geo["over_interp"])
        self.nb = self.oi.shape[1]
        self.corr = corr
        self.nthreads = nthreads

    def oversample(self, f):                       # surface.py:370-375
        return (np.asarray(f).reshape(-1, self.nb) @ self.oi.T).ravel()

    def _c(self, kind, x):
        c = self.corr
        return csr_matvec(c["indptr"], c["indices"], c[kind], x, self.nthreads)

    def pass1(self, tau):
        """(S tau, S' tau) at the sampled rows."""
        w = self.wover * self.oversample(tau)
        pot, grad, _ = p2p(self.nodes, self.over, w[None], None, level=1,
                           nthreads=self.nthreads)
        s = pot[0] / FOUR_PI + self._c("s", tau)
        sp = np.einsum("ik,ik->i", self.normals, grad[0]) / FOUR_PI + self._c("sprime", tau)
        return s, sp

    def pass2(self, tau, mu1, mu2, eta):
        """-tau/4 + S'[mu1] - (S''+D')[mu2] - 2H S'[mu2] + eta at the sampled
        rows; eta = <w, S mu2> / sum w is a global reduction, passed in."""
        wmu1 = self.wover * self.oversample(mu1)
        wmu2 = self.wover * self.oversample(mu2)
        charges = np.stack([wmu1, wmu2, np.zeros_like(wmu1)])
        dipoles = np.zeros((3, len(wmu1), 3))
        dipoles[2] = wmu2[:, None] * self.overn
        pot, grad, hess = p2p(self.nodes, self.over, charges, dipoles, level=2,
                              nthreads=self.nthreads)
        n = self.normals
        sp_mu1 = np.einsum("ik,ik->i", n, grad[0]) / FOUR_PI + self._c("sprime", mu1)
        sp_mu2 = np.einsum("ik,ik->i", n, grad[1]) / FOUR_PI + self._c("sprime", mu2)
        spp = np.einsum("ij,ijk,ik->i", n, hess[1], n) + np.einsum("ik,ik->i", n, grad[2])
        sppdp = spp / FOUR_PI + self._c("spp_plus_dprime", mu2)
        s_mu2 = pot[1] / FOUR_PI + self._c("s", mu2)
        t = np.asarray(tau)[self.rows]
        return -t / 4.0 + sp_mu1 - sppdp - 2.0 * self.curv * sp_mu2 + eta, s_mu2

    def step(self, tau, mu1, mu2, eta=0.0):
        """One sampled apply: pass 1 at the rows, then pass 2 from the given
        full-length mu; returns (result rows, (S tau, S' tau) rows)."""
        s, sp = self.pass1(tau)
        res, _ = self.pass2(tau, mu1, mu2, eta)
        return res, (s, sp)


def synthetic_rows(near_lists, nb, seed=7):
    """CSR rows on the reference's correction pattern for the sampled
    targets (quadrature.py:693-700: nb consecutive columns per near patch,
    patches ascending) with seeded values: TIMING ONLY (the cost of a CSR
    row does not depend on its values)."""
    rng = np.random.default_rng(seed)
    cols = [(np.sort(p)[:, None] * nb + np.arange(nb)[None, :]).ravel() for p in near_lists]
    off = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
    idx = np.concatenate(cols).astype(np.int32)
    out = {"indptr": off, "indices": idx}
    for k in ("s", "sprime", "spp_plus_dprime"):
        out[k] = 1e-3 * rng.standard_normal(len(idx))
    return out
