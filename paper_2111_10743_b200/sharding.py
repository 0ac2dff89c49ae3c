"""Target-sharded operator apply across GPUs.

The apply shards by target rows: rank r owns a contiguous range of patches
(rows [row0, row0 + nrows)); every far sweep still needs ALL sources, so the
intermediate densities are all-gathered between the phases of the apply and
the W-average is all-reduced (lb_opset_apply_phase / lb_opset_phase_exchange).
Collectives are torch.distributed (NCCL over NVLink on the GPUs; gloo in the
CPU tests).  GMRES stays replicated: every rank holds the full Krylov basis
and the apply returns the full result vector (one all-gather of N doubles),
so the Arnoldi arithmetic and its residual history are identical to a single
GPU's.
"""

from __future__ import annotations

import numpy as np

__all__ = ["partition_rows", "allgather_rows", "ShardedApply",
           "ShardedOperatorSet"]


def partition_rows(npatches: int, nb: int, world: int, cost=None):
    """Contiguous patch ranges, one per rank, balanced by `cost` (per-patch
    work, e.g. correction nnz + far rows; uniform when None).  Returns a list
    of (row0, nrows) in target rows (patch-aligned)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if world > npatches:
        raise ValueError(f"cannot give each of {world} ranks a patch "
                         f"({npatches} patches)")
    c = np.ones(npatches) if cost is None else np.asarray(cost, dtype=float)
    cum = np.concatenate([[0.0], np.cumsum(c)])
    bounds = [0]
    for r in range(1, world):
        bounds.append(int(np.searchsorted(cum, cum[-1] * r / world)))
    bounds.append(npatches)
    # every rank owns at least one patch (an empty shard would own nothing
    # yet take part in the reductions): clamp bound r into [r, npatches-world+r]
    bounds = np.array(bounds)
    for r in range(1, world):
        bounds[r] = min(max(bounds[r], bounds[r - 1] + 1), npatches - (world - r))
    return [(int(bounds[r]) * nb, int(bounds[r + 1] - bounds[r]) * nb)
            for r in range(world)]


def allgather_rows(vec, parts, rank, group=None):
    """All-gather the owned rows of a full-length 1-D tensor in place
    (uneven contiguous slices: padded to the largest, then scattered)."""
    import torch
    import torch.distributed as dist
    world = len(parts)
    if world == 1:
        return vec
    m = max(n for _, n in parts)
    r0, nr = parts[rank]
    send = torch.zeros(m, dtype=vec.dtype, device=vec.device)
    send[:nr] = vec[r0:r0 + nr]
    recv = torch.empty(world * m, dtype=vec.dtype, device=vec.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    for q, (q0, qn) in enumerate(parts):
        if q != rank:
            vec[q0:q0 + qn] = recv[q * m:q * m + qn]
    return vec


class ShardedApply:
    """The phase/exchange driver, independent of the compute backend.

    backend must provide: phase(form, p, tau, out), exchange(form, p) ->
    (vector ids, reduce_scalar), work() -> (8, N) tensor, scalar() -> (1,)
    tensor.  The device backend is DeviceOperator (lb_opset_*)."""

    NPHASES = {1: 2, 2: 2, 3: 3}

    def __init__(self, backend, parts, rank, group=None):
        self.backend = backend
        self.parts = parts
        self.rank = rank
        self.group = group

    def apply(self, form: int, tau, out):
        import torch.distributed as dist
        world = len(self.parts)
        for p in range(self.NPHASES[form]):
            self.backend.phase(form, p, tau, out)
            if world == 1:
                continue
            vecs, red = self.backend.exchange(form, p)
            work = self.backend.work()
            for k in vecs:
                allgather_rows(work[k], self.parts, self.rank, self.group)
            if red:
                dist.all_reduce(self.backend.scalar(), group=self.group)
        if world > 1:
            allgather_rows(out, self.parts, self.rank, self.group)
        return out


class _DeviceBackend:
    def __init__(self, dev):
        self.dev = dev

    def phase(self, form, p, tau, out):
        self.dev.apply_phase(form, p, tau, out)

    def exchange(self, form, p):
        return self.dev.phase_exchange(form, p)

    def work(self):
        return self.dev.buffers()[0]

    def scalar(self):
        return self.dev.buffers()[1]


class ShardedOperatorSet:
    """LayerOperatorSet whose applies are split across the ranks of a
    torch.distributed group (one process per GPU).  Same apply/apply_a*
    semantics; results are full vectors on every rank."""

    def __init__(self, disc, formulation, eps, corrections, group=None,
                 far="direct"):
        import torch.distributed as dist
        from . import _lib
        from .operators import (FORMULATIONS, CorrectionSet, DeviceOperator,
                                KernelKind, _FORM_CODE)
        self.formulation = formulation.lower()
        self.eps = float(eps)
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        if not isinstance(corrections, CorrectionSet):
            corrections = CorrectionSet.from_matrices(corrections)
        n = disc.nodes.shape[0]
        nb = disc.over_interp.shape[1] if hasattr(disc, "over_interp") \
            else disc.nodes_per_patch
        npat = n // nb
        ip = corrections.indptr
        cost = (ip[nb::nb] - ip[:-1:nb]) + nb * disc.over_nodes.shape[0] / 50.0
        self.parts = partition_rows(npat, nb, world, cost)
        r0, nr = self.parts[rank]
        kinds = list(FORMULATIONS[self.formulation])
        self.dev = DeviceOperator(disc, corrections, kinds, row0=r0, nrows=nr)
        if far == "fmm":
            # the reference's tree over ALL sources and targets on every rank
            # (deterministic, identical), downward pass + leaf stage only for
            # this rank's target rows: its outputs equal the unsharded FMM's
            from .fmm_plan import FmmPlan
            self._plan = FmmPlan(disc.over_nodes, disc.nodes, self.eps)
            self._plan.set_target_range(r0, r0 + nr)
            self.dev.set_fmm(self._plan)
        elif self.formulation == "a3":
            # fused second sweep; Phi is global (every rank computes it whole)
            from .operators import eta_weights
            self.dev.set_eta_weights(_lib.to_device(eta_weights(disc, corrections)))
        self.driver = ShardedApply(_DeviceBackend(self.dev), self.parts, rank,
                                   group)
        self.rank, self.world, self.n = rank, world, n
        self._code = _FORM_CODE[self.formulation]
        # phi0 = S[1] on the full vector (operators.py:99-100)
        ones = _lib.to_device(np.ones(n))
        phi0 = _lib.zeros((n,))
        self.dev.apply_layer(KernelKind.SINGLE_LAYER, ones, phi0)
        allgather_rows(phi0, self.parts, rank, group)
        self.dev.set_phi0(phi0)
        self._out = _lib.zeros((n,))

    def apply_device(self, tau, out=None):
        from . import _lib
        out = _lib.zeros((self.n,)) if out is None else out
        return self.driver.apply(self._code, tau, out)

    def apply(self, tau):
        from . import _lib
        host = not _lib.is_torch(tau)
        x = _lib.to_device(np.asarray(tau, dtype=float).ravel() if host else tau)
        y = self.apply_device(x)
        return y.cpu().numpy() if host else y
