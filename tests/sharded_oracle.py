"""TEST INFRASTRUCTURE: a CPU (numpy + C oracle) backend for the sharded apply
driver (paper_2111_10743_b200.sharding.ShardedApply), restating the device
phases of csrc/opset.cu (apply_phase) on a row range, so the partitioning and
the phase/exchange protocol can be exercised with gloo on CPU."""

import numpy as np
import torch

import oracle
from oracle.core import FOUR_PI


class OracleShardBackend:
    def __init__(self, bundle, r0, nr):
        self.op = oracle.OracleOperator(bundle, spp="combined")
        self.r0, self.nr = r0, nr
        n = self.op.n
        self.W = torch.zeros((8, n), dtype=torch.float64)
        self.S = torch.zeros(1, dtype=torch.float64)
        self.rows = slice(r0, r0 + nr)

    # far sums for the owned targets only
    def _far(self, charges, dipoles, level):
        op = self.op
        return oracle.p2p(op.nodes[self.rows], op.over, charges, dipoles, level=level)

    def _corr(self, kind, x):
        op = self.op
        ip = op.indptr[self.r0:self.r0 + self.nr + 1]
        return oracle.csr_matvec(ip - ip[0], op.indices[ip[0]:ip[-1]],
                                 op.vals[kind][ip[0]:ip[-1]], x)

    def phase(self, form, p, tau, out):
        op, rows = self.op, self.rows
        tau = tau.numpy()
        n_ = op.normals[rows]
        w = op.weights
        wsum = w.sum()
        if form == 3:
            if p == 0:
                c = op.wover * op.oversample(tau)
                pot, grad, _ = self._far(c[None], None, 1)
                self.W[0, rows] = torch.from_numpy(pot[0] / FOUR_PI + self._corr("s", tau))
                self.W[1, rows] = torch.from_numpy(np.einsum("ik,ik->i", n_, grad[0]) / FOUR_PI
                                                   + self._corr("sprime", tau))
            elif p == 1:
                s_tau, sp_tau = self.W[0].numpy(), self.W[1].numpy()
                c0 = op.wover * op.oversample(sp_tau)
                c1 = op.wover * op.oversample(s_tau)
                pot, grad, _ = self._far(np.stack([c0, c1]), None, 1)
                spp = oracle.spp_far(op.nodes[rows], n_, op.over, op.overn, c1)
                sp_mu1 = np.einsum("ik,ik->i", n_, grad[0]) / FOUR_PI + self._corr("sprime", sp_tau)
                s_mu2 = pot[1] / FOUR_PI + self._corr("s", s_tau)
                sp_mu2 = np.einsum("ik,ik->i", n_, grad[1]) / FOUR_PI + self._corr("sprime", s_tau)
                sppdp = spp / FOUR_PI + self._corr("spp_plus_dprime", s_tau)
                res = -tau[rows] / 4.0 + sp_mu1 - sppdp - 2.0 * op.curv[rows] * sp_mu2
                out[rows] = torch.from_numpy(res)
                self.S[0] = float(np.dot(w[rows], s_mu2)) / wsum
            else:
                out[rows] += self.S[0]
            return
        raise NotImplementedError(form)

    def exchange(self, form, p):
        if form == 3:
            return ([0, 1], False) if p == 0 else ([], p == 1)
        return (list(range(2 if form == 2 else 3)), True) if p == 0 else ([], False)

    def work(self):
        return self.W

    def scalar(self):
        return self.S
