"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
FOUR_PI = 4.0 * np.pi            # kernels.py:16

_lib = None
_P = ctypes.c_void_p


def build(force=False):
    src = os.path.join(HERE, "p2p_oracle.c")
    if force or not os.path.exists(LIB) or \
            os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "-B", "liboracle.so"],
                       check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        I64, I32, U32 = ctypes.c_int64, ctypes.c_int, ctypes.c_uint32
        L.oracle_p2p.argtypes = [_P, I64, _P, I64, _P, _P, I32, U32, U32, I32,
                                 _P, _P, _P, I32, I32]
        L.oracle_p2p_grouped.argtypes = [_P, _P, _P, I64, _P, _P, _P, _P, I64,
                                         I32, U32, U32, I32, I64, _P, _P, _P,
                                         I32]
        L.oracle_csr_matvec.argtypes = [_P, _P, _P, I64, _P, _P, I32, I32]
        L.oracle_max_threads.argtypes = []
        L.oracle_spp_far.argtypes = [_P, _P, I64, _P, _P, _P, I64, _P, I32]
        _lib = L
    return _lib


def _p(a):
    return _P(0) if a is None else a.ctypes.data_as(_P)


def _mask(flags):
    m = 0
    for i, f in enumerate(np.asarray(flags, dtype=bool).ravel()):
        if f:
            m |= 1 << i
    return m


def max_threads():
    return int(lib().oracle_max_threads())


def p2p(tgt, src, charges=None, dipoles=None, level=1, cmask=None,
        dmask=None, nthreads=0):
    """All-pairs direct sum (evaluate_direct, fmm.py:215-222); returns
    (pot, grad|None, hess|None) in the reference layouts."""
    tgt = np.ascontiguousarray(tgt, dtype=float)
    src = np.ascontiguousarray(src, dtype=float)
    nd = (charges if charges is not None else dipoles).shape[0]
    if charges is not None:
        charges = np.ascontiguousarray(charges, dtype=float)
    if dipoles is not None:
        dipoles = np.ascontiguousarray(dipoles, dtype=float)
    if cmask is None:
        cmask = _mask(np.abs(charges).max(axis=1) > 0) if charges is not None \
            and charges.size else 0
    if dmask is None:
        dmask = _mask(np.abs(dipoles).max(axis=(1, 2)) > 0) \
            if dipoles is not None and dipoles.size else 0
    nt = tgt.shape[0]
    pot = np.zeros((nd, nt))
    grad = np.zeros((nd, nt, 3)) if level >= 1 else None
    hess = np.zeros((nd, nt, 3, 3)) if level >= 2 else None
    rc = lib().oracle_p2p(_p(tgt), nt, _p(src), src.shape[0], _p(charges),
                          _p(dipoles), nd, cmask, dmask, level, _p(pot),
                          _p(grad), _p(hess), 0, nthreads)
    assert rc == 0
    return pot, grad, hess


def p2p_grouped(t_xyz, t_out, t_off, s_xyz, s_c, s_v, s_off, use_c, use_d,
                level, nd, ntargets, nthreads=0):
    """grouped_direct + run_grouped_direct (_pointsum.py:19-114)."""
    c = lambda a, dt=float: np.ascontiguousarray(a, dtype=dt)  # noqa: E731
    t_xyz, s_xyz = c(t_xyz), c(s_xyz)
    t_out, t_off, s_off = c(t_out, np.int64), c(t_off, np.int64), \
        c(s_off, np.int64)
    s_c, s_v = c(s_c), c(s_v)
    pot = np.zeros((nd, ntargets))
    grad = np.zeros((nd, ntargets, 3))
    hess = np.zeros((nd, ntargets, 3, 3))
    rc = lib().oracle_p2p_grouped(
        _p(t_xyz), _p(t_out), _p(t_off), len(t_off) - 1, _p(s_xyz), _p(s_c),
        _p(s_v), _p(s_off), s_xyz.shape[0], nd, _mask(use_c), _mask(use_d),
        level, ntargets, _p(pot), _p(grad), _p(hess), nthreads)
    assert rc == 0
    return pot, grad, hess


def csr_matvec(indptr, indices, data, x, nthreads=0):
    """y = A x for scipy-CSR arrays (operators.py:155 `corr(kind) @ tau`)."""
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    data = np.ascontiguousarray(data, dtype=float)
    x = np.ascontiguousarray(x, dtype=float)
    y = np.zeros(len(indptr) - 1)
    lib().oracle_csr_matvec(_p(indptr), _p(indices), _p(data), len(y), _p(x),
                            _p(y), 0, nthreads)
    return y


def spp_far(x, nx, y, ny, c, nthreads=0):
    """Combined-form S''+D' far sum (kernels.py:60-67 kernel, no 4 pi)."""
    x, nx, y, ny, c = (np.ascontiguousarray(a, dtype=float)
                       for a in (x, nx, y, ny, c))
    out = np.zeros(x.shape[0])
    lib().oracle_spp_far(_p(x), _p(nx), x.shape[0], _p(y), _p(ny), _p(c),
                         y.shape[0], _p(out), nthreads)
    return out
