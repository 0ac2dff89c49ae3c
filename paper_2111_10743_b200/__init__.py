"""B200-native (sm_100a) implementation of the GMRES operator-apply hot path of
the reference Laplace-Beltrami package `lapbel` (arXiv:2111.10743).

The public names mirror `lapbel/__init__.py:37-50` for the hot path: the point
sums (FmmSources, FmmResult, evaluate_direct, evaluate_fmm, FmmPlan), the
operator set (LayerOperatorSet, DensityVector), the solver (gmres,
solve_laplace_beltrami, SolveConfig, SolveReport) and, widening into
SURVEY §8(f) #1, the near-correction build (build_near_map,
compute_corrections) and, §8(f) #4, the lbmesh reader/writer with the
device geometry build (read_mesh, write_mesh, build_from_coefficients).  All arithmetic runs in
libb200lb.so; there is no CPU fallback.
"""

__version__ = "0.1.0"

from .fmm import (FmmCapacityError, FmmPlan, FmmResult, FmmSources,
                  evaluate_direct, evaluate_fmm, order_for_eps)
from ._pointsum import run_grouped_direct
from .operators import (FORMULATIONS, CorrectionSet, DensityVector, Geometry,
                        KernelKind, LayerOperatorSet, apply_layer)
from .solver import (GmresBreakdown, SolveConfig, SolveReport, gmres,
                     solve_laplace_beltrami)
from .quadrature import (AdaptiveDepthError, NearMap, NearMapCapError,
                         build_near_map, compute_corrections)
from .simplex import ReferenceElement, reference_element
from .surface import (DegeneratePatchError, SurfaceDiscretization,
                      build_from_coefficients)
from .meshio import read_mesh, write_mesh

__all__ = [
    "FmmSources", "FmmResult", "FmmCapacityError", "FmmPlan",
    "evaluate_direct", "evaluate_fmm", "order_for_eps", "run_grouped_direct",
    "KernelKind", "FORMULATIONS", "DensityVector", "Geometry", "CorrectionSet",
    "LayerOperatorSet", "apply_layer", "SolveConfig", "SolveReport",
    "GmresBreakdown", "gmres", "solve_laplace_beltrami",
    "NearMap", "NearMapCapError", "AdaptiveDepthError", "build_near_map",
    "compute_corrections", "ReferenceElement", "reference_element",
    "DegeneratePatchError", "SurfaceDiscretization", "build_from_coefficients",
    "read_mesh", "write_mesh",
]
