"""Grouped multi-density point sums: the drop-in for lapbel._pointsum
(`_pointsum.py:92-114`), running the CUDA grouped kernel (csrc/p2p.cu)."""

from __future__ import annotations

import numpy as np

from . import _lib


def run_grouped_direct(t_xyz, t_out, t_off, s_xyz, s_c, s_v, s_off,
                       use_c, use_d, want, nd, ntargets):
    """Allocate zeroed outputs, accumulate every group's sums, return a dict
    {"pot": (nd,ntargets), "grad": (nd,ntargets,3), "hess": (nd,ntargets,3,3)}
    with the Hessian symmetric (_pointsum.py:92-114).  Level 0/1/2 follows
    `want` exactly as the reference."""
    t = _lib.require_cuda()
    host = not _lib.is_torch(t_xyz)
    level = 2 if "hess" in want else (1 if "grad" in want else 0)
    dev = _lib.to_device
    txyz = dev(t_xyz)
    tout = dev(t_out, t.int64)
    toff = dev(t_off, t.int64)
    sxyz = dev(s_xyz)
    soff = dev(s_off, t.int64)
    cm = _lib.mask_of(use_c)
    dm = _lib.mask_of(use_d)
    sc = dev(s_c) if cm and s_c is not None else None
    sv = dev(s_v) if dm and s_v is not None else None
    cm = cm if sc is not None else 0
    dm = dm if sv is not None else 0
    pot = _lib.zeros((nd, ntargets))
    grad = _lib.zeros((nd, ntargets, 3)) if level >= 1 else _lib.zeros((nd, 0, 3))
    hess = _lib.zeros((nd, ntargets, 3, 3)) if level >= 2 \
        else _lib.zeros((nd, 0, 3, 3))
    ngroups = int(toff.shape[0]) - 1
    _lib.call("lb_p2p_grouped", _lib.ptr(txyz), _lib.ptr(tout), _lib.ptr(toff),
              ngroups, txyz.shape[0], _lib.ptr(sxyz), _lib.ptr(sc),
              _lib.ptr(sv), _lib.ptr(soff), sxyz.shape[0], nd, cm, dm, level,
              ntargets, _lib.ptr(pot), _lib.ptr(grad), _lib.ptr(hess),
              _lib.stream_handle())

    def conv(x):
        return x.cpu().numpy() if host else x
    out = {"pot": conv(pot)}
    if "grad" in want:
        out["grad"] = conv(grad)
    if "hess" in want:
        out["hess"] = conv(hess)
    return out


__all__ = ["run_grouped_direct"]
_ = np
