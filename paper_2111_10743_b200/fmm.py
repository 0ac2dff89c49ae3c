"""Multi-density 1/r point sums on the B200: the drop-in for lapbel.fmm.

Same names, argument meaning, layouts and error behaviour as the reference
(`/root/reference/pkg/src/lapbel/fmm.py`): the kernel is
    u_l(x) = sum_j c_{l,j}/|x - s_j| - v_{l,j} . grad_x 1/|x - s_j|
WITHOUT the 1/(4 pi) (fmm.py:3-9), coincident pairs contribute nothing
(fmm.py:136-141), pot (nd,Nt), grad (nd,Nt,3), hess (nd,Nt,3,3) symmetric.

Every evaluation runs in libb200lb.so (hand-written sm_100a kernels); inputs
may be numpy arrays (results come back as numpy, like the reference) or CUDA
torch tensors (results stay on the device).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import FmmCapacityError

__all__ = [
    "FmmSources",
    "FmmResult",
    "FmmCapacityError",
    "evaluate_direct",
    "evaluate_fmm",
    "FmmPlan",
    "order_for_eps",
]


# ---------------------------------------------------------------------------
# sources / results (fmm.py:47-123)


def _as_float_array(a):
    if _lib.is_torch(a):
        return a.to(dtype=_lib.torch().float64).contiguous()
    return np.ascontiguousarray(a, dtype=float)


def _amax(a, axis):
    if _lib.is_torch(a):
        t = _lib.torch()
        return t.amax(t.abs(a), dim=axis).cpu().numpy()
    return np.abs(a).max(axis=axis)


@dataclass
class FmmSources:
    """Point sources with nd densities of charges and/or dipole vectors
    (fmm.py:47-103): positions (M,3), charges (nd,M), dipoles (nd,M,3)."""

    positions: object
    charges: object = None
    dipoles: object = None

    def __post_init__(self):
        self.positions = _as_float_array(self.positions)
        if self.positions.ndim != 2 or self.positions.shape[1] != 3:
            raise ValueError("positions must have shape (M, 3)")
        m = self.positions.shape[0]
        if self.charges is None and self.dipoles is None:
            raise ValueError("need charges and/or dipoles")
        if self.charges is not None:
            self.charges = _as_float_array(self.charges)
            if self.charges.ndim == 1:
                self.charges = self.charges[None, :]
            if self.charges.shape[1] != m:
                raise ValueError("charges must have shape (nd, M)")
        if self.dipoles is not None:
            self.dipoles = _as_float_array(self.dipoles)
            if self.dipoles.ndim == 2:
                self.dipoles = self.dipoles[None, :, :]
            if tuple(self.dipoles.shape[1:]) != (m, 3):
                raise ValueError("dipoles must have shape (nd, M, 3)")
        if self.charges is not None and self.dipoles is not None \
                and self.charges.shape[0] != self.dipoles.shape[0]:
            raise ValueError("charge/dipole density counts differ")

    @property
    def nsources(self) -> int:
        return self.positions.shape[0]

    @property
    def nd(self) -> int:
        if self.charges is not None:
            return self.charges.shape[0]
        return self.dipoles.shape[0]

    @property
    def charge_active(self) -> np.ndarray:
        if self.charges is None:
            return np.zeros(self.nd, dtype=bool)
        if self.nsources == 0:
            return np.zeros(self.nd, dtype=bool)
        return _amax(self.charges, 1) > 0.0

    @property
    def dipole_active(self) -> np.ndarray:
        if self.dipoles is None:
            return np.zeros(self.nd, dtype=bool)
        if self.nsources == 0:
            return np.zeros(self.nd, dtype=bool)
        return _amax(self.dipoles, (1, 2)) > 0.0


@dataclass
class FmmResult:
    """Potentials (nd, Nt), and gradients (nd, Nt, 3) / Hessians
    (nd, Nt, 3, 3) when requested (fmm.py:106-113)."""

    pot: object
    grad: object = None
    hess: object = None


def _parse_outputs(outputs):
    """fmm.py:116-123."""
    want = set(outputs)
    bad = want - {"pot", "grad", "hess"}
    if bad:
        raise ValueError(f"unknown outputs {sorted(bad)}")
    if "pot" not in want:
        want.add("pot")
    return want


def _level(want) -> int:
    return 2 if "hess" in want else (1 if "grad" in want else 0)


def _alloc_device_result(nd, nt, level):
    pot = _lib.empty((nd, nt))
    grad = _lib.empty((nd, nt, 3)) if level >= 1 else None
    hess = _lib.empty((nd, nt, 3, 3)) if level >= 2 else None
    return pot, grad, hess


def _finish(want, pot, grad, hess, host: bool):
    def conv(x):
        return x.cpu().numpy() if host and x is not None else x
    return FmmResult(pot=conv(pot),
                     grad=conv(grad) if "grad" in want else None,
                     hess=conv(hess) if "hess" in want else None)


# ---------------------------------------------------------------------------
# direct summation (fmm.py:130-222)


def p2p_device(tgt, src, charges, dipoles, nd, cmask, dmask, level,
               pot, grad=None, hess=None, accumulate=False, stream=None):
    """Thin wrapper of lb_p2p on device tensors (no shape conversion)."""
    _lib.call("lb_p2p", _lib.ptr(tgt), tgt.shape[0], _lib.ptr(src),
              src.shape[0], _lib.ptr(charges), _lib.ptr(dipoles), nd, cmask,
              dmask, level, _lib.ptr(pot), _lib.ptr(grad), _lib.ptr(hess),
              int(bool(accumulate)), _lib.stream_handle(stream))


def evaluate_direct(sources: FmmSources, targets, outputs=("pot",)) -> FmmResult:
    """Exact O(M Nt) summation; coincident source/target pairs are skipped
    (fmm.py:215-222).  Runs the tiled fp64 P2P kernel (csrc/p2p.cu)."""
    want = _parse_outputs(outputs)
    host = not _lib.is_torch(targets)
    tgt = _lib.to_device(targets)
    if tgt.ndim != 2 or tgt.shape[1] != 3:
        raise ValueError("targets must have shape (Nt, 3)")
    nd = sources.nd
    level = _level(want)
    cm = _lib.mask_of(sources.charge_active)
    dm = _lib.mask_of(sources.dipole_active)
    src = _lib.to_device(sources.positions)
    ch = _lib.to_device(sources.charges) if cm else None
    dp = _lib.to_device(sources.dipoles) if dm else None
    pot, grad, hess = _alloc_device_result(nd, tgt.shape[0], level)
    p2p_device(tgt, src, ch, dp, nd, cm, dm, level, pot, grad, hess)
    return _finish(want, pot, grad, hess, host)


from .fmm_plan import FmmPlan, evaluate_fmm, order_for_eps  # noqa: E402
