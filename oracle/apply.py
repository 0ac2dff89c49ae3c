"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Numpy restatement of the operator applies and GMRES of the reference:
  apply_layer      operators.py:126-155
  apply_a1/a2/a3   operators.py:161-266 (the use_fmm=False path: the far
                   field is the exact direct sum, here oracle.p2p in C)
  gmres            solver.py:48-103
  solve            solver.py:106-154
Inputs are plain arrays (a "bundle" dict as written by scripts/make_golden.py).
"""

from __future__ import annotations

import numpy as np

from .core import FOUR_PI, csr_matvec, p2p, spp_far

KINDS = ("s", "d", "sprime", "grads1", "grads2", "grads3", "spp_plus_dprime")
FORMS = {"a1": ("s", "grads1", "grads2", "grads3"),
         "a2": ("s", "d", "sprime", "spp_plus_dprime"),
         "a3": ("s", "sprime", "spp_plus_dprime")}


class OracleOperator:
    def __init__(self, b, nthreads=0, spp="separate"):
        """spp="separate" evaluates the S''+D' far sum exactly as the
        reference (n.H.n + n.grad of a dipole, operators.py:257-259);
        spp="combined" uses the cancellation-free kernel of kernels.py:60-67
        (what the CUDA path computes)."""
        self.b = b
        self.spp = spp
        self.nthreads = nthreads
        self.nodes = np.asarray(b["nodes"])
        self.normals = np.asarray(b["normals"])
        self.weights = np.asarray(b["weights"])
        self.curv = np.asarray(b["curvature"])
        self.over = np.asarray(b["over_nodes"])
        self.overn = np.asarray(b["over_normals"])
        self.wover = np.asarray(b["over_weights"])
        self.oi = np.asarray(b["over_interp"])
        self.indptr = np.asarray(b["corr_indptr"])
        self.indices = np.asarray(b["corr_indices"])
        self.vals = {k: np.asarray(b["corr_" + k]) for k in KINDS
                     if "corr_" + k in b}
        self.nb = self.oi.shape[1]
        self.n = self.nodes.shape[0]
        self.phi0 = self.apply_layer("s", np.ones(self.n))

    # surface.py:370-375
    def oversample(self, f):
        return (np.asarray(f).reshape(-1, self.nb) @ self.oi.T).ravel()

    def corr(self, kind, x):
        return csr_matvec(self.indptr, self.indices, self.vals[kind], x,
                          self.nthreads)

    # operators.py:103-114 (use_fmm=False): direct sums, no 4 pi
    def far(self, charges, dipoles, level):
        return p2p(self.nodes, self.over, charges, dipoles, level=level,
                   nthreads=self.nthreads)

    def spp_sum(self, c):
        return spp_far(self.nodes, self.normals, self.over, self.overn, c,
                       self.nthreads)

    def apply_layer(self, kind, tau):
        w = self.wover * self.oversample(tau)
        n = self.normals
        if kind in ("s", "sprime", "grads1", "grads2", "grads3"):
            pot, grad, _ = self.far(w[None], None, 0 if kind == "s" else 1)
            if kind == "s":
                far = pot[0]
            elif kind == "sprime":
                far = np.einsum("ik,ik->i", n, grad[0])
            else:
                far = grad[0][:, int(kind[-1]) - 1]
        elif kind == "d":
            pot, _, _ = self.far(None, (w[:, None] * self.overn)[None], 0)
            far = pot[0]
        elif kind == "spp_plus_dprime" and self.spp == "combined":
            far = self.spp_sum(w)
        elif kind == "spp_plus_dprime":
            dip = (w[:, None] * self.overn)[None]
            _, grad, hess = self.far(np.vstack([w[None], np.zeros_like(w)[None]]),
                                     np.concatenate([np.zeros_like(dip), dip]), 2)
            far = np.einsum("ij,ijk,ik->i", n, hess[0], n) \
                + np.einsum("ik,ik->i", n, grad[1])
        else:
            raise ValueError(kind)
        return far / FOUR_PI + self.corr(kind, tau)

    def apply_a1(self, tau):
        b = self.b
        w = self.wover * self.oversample(tau)
        pot, grad, _ = self.far(w[None], None, 1)
        s_tau = pot[0] / FOUR_PI + self.corr("s", tau)
        grad_s = grad[0] / FOUR_PI
        grad_s += np.column_stack([self.corr(k, tau)
                                   for k in ("grads1", "grads2", "grads3")])
        tu, tv, gi = b["tangents_u"], b["tangents_v"], b["inv_metric"]
        gu = np.einsum("ik,ik->i", grad_s, tu)
        gv = np.einsum("ik,ik->i", grad_s, tv)
        a = gi[:, 0, 0] * gu + gi[:, 0, 1] * gv
        bb = gi[:, 1, 0] * gu + gi[:, 1, 1] * gv
        mu = a[:, None] * tu + bb[:, None] * tv
        charges = np.stack([self.wover * self.oversample(mu[:, l])
                            for l in range(3)])
        _, grad2, _ = self.far(charges, None, 1)
        div = np.zeros(self.n)
        for l, kind in enumerate(("grads1", "grads2", "grads3")):
            div += grad2[l][:, l] / FOUR_PI + self.corr(kind, mu[:, l])
        eta = float(np.dot(s_tau, self.weights) / self.weights.sum())
        return div + eta * self.phi0

    def apply_a2(self, tau):
        w = self.wover * self.oversample(tau)
        dip = w[:, None] * self.overn
        pot, grad, hess = self.far(np.stack([w, np.zeros_like(w)]),
                                   np.stack([np.zeros_like(dip), dip]), 2)
        n = self.normals
        s_tau = pot[0] / FOUR_PI + self.corr("s", tau)
        d_tau = pot[1] / FOUR_PI + self.corr("d", tau)
        sp_tau = np.einsum("ik,ik->i", n, grad[0]) / FOUR_PI \
            + self.corr("sprime", tau)
        if self.spp == "combined":
            spp = self.spp_sum(w)
        else:
            spp = np.einsum("ij,ijk,ik->i", n, hess[0], n) \
                + np.einsum("ik,ik->i", n, grad[1])
        sppdp_tau = spp / FOUR_PI + self.corr("spp_plus_dprime", tau)
        ws = float(np.dot(self.weights, s_tau) / self.weights.sum())
        mu1 = d_tau
        mu2 = -sppdp_tau - 2.0 * self.curv * sp_tau + ws
        wmu1 = self.wover * self.oversample(mu1)
        wmu2 = self.wover * self.oversample(mu2)
        charges2 = np.stack([np.zeros_like(wmu2), wmu2])
        dipoles2 = np.stack([wmu1[:, None] * self.overn,
                             np.zeros((len(wmu1), 3))])
        pot2, _, _ = self.far(charges2, dipoles2, 0)
        d_mu1 = pot2[0] / FOUR_PI + self.corr("d", mu1)
        s_mu2 = pot2[1] / FOUR_PI + self.corr("s", mu2)
        return -tau / 4.0 + s_mu2 + d_mu1

    def apply_a3(self, tau):
        w = self.wover * self.oversample(tau)
        pot, grad, _ = self.far(w[None], None, 1)
        n = self.normals
        s_tau = pot[0] / FOUR_PI + self.corr("s", tau)
        sp_tau = np.einsum("ik,ik->i", n, grad[0]) / FOUR_PI \
            + self.corr("sprime", tau)
        mu1, mu2 = sp_tau, s_tau
        wmu1 = self.wover * self.oversample(mu1)
        wmu2 = self.wover * self.oversample(mu2)
        charges2 = np.stack([wmu1, wmu2, np.zeros_like(wmu1)])
        dipoles2 = np.zeros((3, len(wmu1), 3))
        dipoles2[2] = wmu2[:, None] * self.overn
        pot2, grad2, hess2 = self.far(charges2, dipoles2, 2)
        sp_mu1 = np.einsum("ik,ik->i", n, grad2[0]) / FOUR_PI \
            + self.corr("sprime", mu1)
        s_mu2 = pot2[1] / FOUR_PI + self.corr("s", mu2)
        sp_mu2 = np.einsum("ik,ik->i", n, grad2[1]) / FOUR_PI \
            + self.corr("sprime", mu2)
        if self.spp == "combined":
            spp = self.spp_sum(wmu2)
        else:
            spp = np.einsum("ij,ijk,ik->i", n, hess2[1], n) \
                + np.einsum("ik,ik->i", n, grad2[2])
        sppdp_mu2 = spp / FOUR_PI + self.corr("spp_plus_dprime", mu2)
        eta = float(np.dot(self.weights, s_mu2) / self.weights.sum())
        return -tau / 4.0 + sp_mu1 - sppdp_mu2 \
            - 2.0 * self.curv * sp_mu2 + eta

    def apply(self, form, tau):
        return getattr(self, "apply_" + form)(tau)

    def evaluate_solution(self, form, sigma):
        u = self.apply_layer("s", sigma)
        if form == "a3":
            u = self.apply_layer("s", u)
        return u


def gmres(apply_fn, rhs, tol=1e-8, max_iter=100):
    """solver.py:48-103, restated."""
    rhs = np.asarray(rhs, dtype=float)
    n = rhs.size
    bnorm = float(np.linalg.norm(rhs))
    if bnorm == 0.0:
        return np.zeros(n), [0.0], True
    max_iter = min(max_iter, n)
    q = np.zeros((max_iter + 1, n))
    h = np.zeros((max_iter + 1, max_iter))
    cs = np.zeros(max_iter)
    sn = np.zeros(max_iter)
    g = np.zeros(max_iter + 1)
    g[0] = bnorm
    q[0] = rhs / bnorm
    history = []
    converged = False
    k_used = 0
    for k in range(max_iter):
        v = np.array(apply_fn(q[k]), dtype=float, copy=True)
        for j in range(k + 1):
            h[j, k] = np.dot(q[j], v)
            v -= h[j, k] * q[j]
        h[k + 1, k] = np.linalg.norm(v)
        happy = h[k + 1, k] <= 1e-14 * bnorm
        if not happy:
            q[k + 1] = v / h[k + 1, k]
        for j in range(k):
            t = cs[j] * h[j, k] + sn[j] * h[j + 1, k]
            h[j + 1, k] = -sn[j] * h[j, k] + cs[j] * h[j + 1, k]
            h[j, k] = t
        denom = np.hypot(h[k, k], h[k + 1, k])
        if denom == 0.0:
            raise RuntimeError("GMRES breakdown")
        cs[k] = h[k, k] / denom
        sn[k] = h[k + 1, k] / denom
        h[k, k] = denom
        h[k + 1, k] = 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        history.append(abs(g[k + 1]) / bnorm)
        k_used = k + 1
        if history[-1] <= tol or happy:
            converged = True
            break
    y = np.linalg.solve(np.triu(h[:k_used, :k_used]), g[:k_used])
    return y @ q[:k_used], history, converged


def solve(op: OracleOperator, form, f, eps_gmres=1e-10, max_iter=100):
    """solver.py:106-154 restated; returns (sigma, u, history)."""
    w = op.weights
    f = np.asarray(f, dtype=float)
    f = f - float(np.dot(w, f)) / float(w.sum())
    rhs = op.apply_layer("s", f) if form in ("a1", "a2") else f
    sigma, hist, conv = gmres(lambda t: op.apply(form, t), rhs, eps_gmres,
                              max_iter)
    return sigma, op.evaluate_solution(form, sigma), hist
