"""FmmPlan / evaluate_fmm / order_for_eps (fmm.py:357-382, 722-1011)."""

from __future__ import annotations


def order_for_eps(eps: float):
    """(representation, size, separation buffer) for a requested tolerance
    (fmm.py:357-382, same thresholds)."""
    if eps >= 1e-3:
        return "surface", 5, 1
    if eps >= 1e-4:
        return "surface", 6, 1
    if eps >= 1e-5:
        return "surface", 7, 1
    if eps >= 1e-6:
        return "surface", 8, 1
    if eps >= 2e-7:
        return "surface", 9, 1
    if eps >= 3e-8:
        return "surface", 10, 1
    if eps >= 1e-9:
        return "grid", 9, 2
    return "grid", 11, 2


class FmmPlan:  # pragma: no cover - replaced by the GPU plan
    def __init__(self, *a, **k):
        raise NotImplementedError("GPU FmmPlan not built yet")


def evaluate_fmm(*a, **k):  # pragma: no cover
    raise NotImplementedError("GPU FMM not built yet")
