"""ctypes binding of libb200lb.so (the C ABI declared in include/lapbel_b200.h)
plus the small amount of device plumbing the Python mirror needs.

There is deliberately no CPU fallback: if the library or a CUDA device is
missing, every entry point raises.  torch is used only for device memory and
streams.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libb200lb.so")

LB_OK = 0
LB_ERR_SHAPE = 1
LB_ERR_EPS = 2
LB_ERR_CAPACITY = 3
LB_ERR_CUDA = 4
LB_ERR_NCCL = 5
LB_ERR_ARG = 6
LB_ERR_KEY = 7
LB_ERR_BREAKDOWN = 8
LB_ERR_DEPTH = 9
LB_ERR_NEARCAP = 10

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_U32 = ctypes.c_uint32
_F64 = ctypes.c_double

# name -> argtypes (restype is always int / lb_status unless listed in _RES)
SIGNATURES = {
    "lb_abi_version": [],
    "lb_last_error_string": [],
    "lb_device_info": [_P, _P, _P],
    "lb_graph_kernel_nodes": [_P, _P, _P],
    "lb_p2p": [_P, _I64, _P, _I64, _P, _P, _I32, _U32, _U32, _I32, _P, _P, _P,
               _I32, _P],
    "lb_p2p_grouped": [_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _I64, _I32,
                       _U32, _U32, _I32, _I64, _P, _P, _P, _P],
    "lb_opset_create": [_P, _P],
    "lb_opset_destroy": [_P],
    "lb_opset_set_phi0": [_P, _P],
    "lb_opset_set_eta_weights": [_P, _P],
    "lb_opset_set_fmm_a3": [_P, _I32],
    "lb_opset_set_fmm": [_P, _P],
    "lb_opset_apply_phase": [_P, _I32, _I32, _P, _P, _P],
    "lb_opset_phase_exchange": [_P, _I32, _I32, _P, _P, _P],
    "lb_opset_buffers": [_P, _P, _P, _P, _P],
    "lb_opset_set_timing": [_P, _I32],
    "lb_opset_stage_times": [_P, _P],
    "lb_opset_apply": [_P, _I32, _P, _P, _P],
    "lb_opset_apply_layer": [_P, _I32, _P, _P, _P],
    "lb_opset_last_scalar": [_P, _P],
    "lb_opset_time_far": [_P, _I32, _I32, _P, _P],
    "lb_csr_spmv": [_P, _P, _I64, _I32, _P, _P, _P, _I32, _P],
    "lb_arnoldi_mgs": [_P, _I64, _I32, _I64, _P, _P, _P],
    "lb_combine_rows": [_P, _I64, _I32, _I64, _P, _P, _P],
    "lb_dot": [_P, _P, _I64, _P, _P],
    "lb_nrm2": [_P, _I64, _P, _P],
    "lb_scale_inv": [_P, _P, _I64, _P, _P],
    "lb_fmm_plan_create": [_P, _I64, _P, _I64, _I32, _I32, _I32, _P],
    "lb_fmm_plan_destroy": [_P],
    "lb_fmm_plan_info": [_P, _P, _P],
    "lb_fmm_plan_export": [_P, _I32, _P],
    "lb_fmm_plan_set_operators": [_P, _P],
    "lb_fmm_apply": [_P, _P, _P, _I32, _U32, _U32, _I32, _P, _P, _P, _P],
    "lb_fmm_plan_set_timing": [_P, _I32],
    "lb_fmm_plan_set_m2l": [_P, _I32],
    "lb_fmm_plan_set_xw": [_P, _I32],
    "lb_fmm_plan_set_m2l_factors": [_P, _P, _P, _P],
    "lb_fmm_plan_set_target_range": [_P, _I64, _I64],
    "lb_fmm_plan_set_source_range": [_P, _I64, _I64],
    "lb_fmm_plan_set_upward_hook": [_P, _P, _P],
    "lb_near_map_count": [_P, _I64, _P, _P, _I64, _P, _P, _P],
    "lb_near_map_fill": [_P, _I64, _P, _P, _I64, _P, _P, _P, _P],
    "lb_corrections_build": [_P, _P],
    "lb_geom_build": [_P, _P],
    "lb_fmm_stage_times": [_P, _P],
    "lb_fmm_setup_times": [_P, _P],
    "lb_probe_dfma": [_P, _I32, _I32, _P],
    "lb_probe_dmma": [_P, _I32, _I32, _P],
    "lb_probe_dmma_operands": [_P, _I32, _I32, _I32, _P],
    "lb_probe_mixed": [_P, _I32, _I32, _I32, _I32, _P],
    "lb_probe_read_rows": [_P, _P, _I64, _I64, _P, _P],
    "lb_dgemm_cols": [_P, _I32, _I32, _I32, _P, _I64, _P, _P, _P, _I64, _P, _I64,
                      ctypes.c_double, _I32, _P],
    "lb_probe_rsqrt": [_P, _P, _I64, _I32, _P],
}
_RES = {"lb_last_error_string": ctypes.c_char_p}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryMissing(
            f"{path} is not built; run `python -m paper_2111_10743_b200._build`"
            " (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RES.get(name, ctypes.c_int)
    _lib = lib
    return lib


def exported_symbols():
    return sorted(SIGNATURES)


# ---------------------------------------------------------------------------
# status -> reference exception types

class FmmCapacityError(RuntimeError):
    """Pathological point clustering: octree refinement cap exceeded
    (fmm.py:39-40)."""


class AdaptiveDepthError(RuntimeError):
    """Adaptive subdivision hit the depth cap (quadrature.py:62-63)."""


class NearMapCapError(RuntimeError):
    """A target's near set exceeded the patch cap (quadrature.py:58-59)."""


class GmresBreakdown(RuntimeError):
    """Arnoldi norm underflow that is not a happy breakdown (solver.py:18)."""


def check(status: int, what: str = ""):
    if status == LB_OK:
        return
    msg = load().lb_last_error_string().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status in (LB_ERR_SHAPE, LB_ERR_ARG, LB_ERR_EPS):
        raise ValueError(text)
    if status == LB_ERR_CAPACITY:
        raise FmmCapacityError(text)
    if status == LB_ERR_KEY:
        raise KeyError(text)
    if status == LB_ERR_BREAKDOWN:
        raise GmresBreakdown(text)
    if status == LB_ERR_DEPTH:
        raise AdaptiveDepthError(text)
    if status == LB_ERR_NEARCAP:
        raise NearMapCapError(text)
    raise RuntimeError(f"libb200lb error {status}: {text}")


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)


# ---------------------------------------------------------------------------
# device plumbing (torch = memory + streams only)

def torch():
    import torch as _torch
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2111_10743_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    load()
    return t


def stream_handle(stream=None):
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return _P(s.cuda_stream)


def ptr(x):
    if x is None:
        return _P(0)
    return _P(x.data_ptr())


def to_device(a, dtype=None):
    """numpy/torch -> contiguous CUDA tensor (float64 by default)."""
    t = require_cuda()
    dt = dtype or t.float64
    if isinstance(a, t.Tensor):
        return a.to(device="cuda", dtype=dt).contiguous()
    arr = np.ascontiguousarray(a)
    return t.from_numpy(arr).to(device="cuda", dtype=dt).contiguous()


def empty(shape, dtype=None):
    t = require_cuda()
    return t.empty(shape, dtype=dtype or t.float64, device="cuda")


def zeros(shape, dtype=None):
    t = require_cuda()
    return t.zeros(shape, dtype=dtype or t.float64, device="cuda")


def is_torch(a) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(a, _t.Tensor)


def mask_of(flags) -> int:
    m = 0
    for i, f in enumerate(np.asarray(flags, dtype=bool).ravel()):
        if f:
            m |= 1 << i
    return m
