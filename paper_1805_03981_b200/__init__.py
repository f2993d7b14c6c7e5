"""B200-native DG-acoustics hot path (arXiv 1805.03981 reference `wavekernel`).

Drop-in GPU replacements for the reference operator and steppers; see
DESIGN.md.  Kernels are hand-written FP64 CUDA for sm_100a behind the C ABI
in include/wavekernel_b200.h (library: libwk_b200.so, built in-tree).
"""

from .operator import AcousticOperator, FluxParams, StateVector, hdg_flux
from .stepping import (LSRK45, LSRK59, RK4_CLASSIC, SchemeConfig, DeviceStepper,
                       CourantSearchError, ader_step, advance, compute_dt,
                       find_critical_courant, lsrk_step, make_stepper, rk_step,
                       state_norm, tck_evaluate)
from .analytic import exact_pressure_norm, initial_state, l2_pressure_error
from .mesh import (GeometryError, Material, Mesh, affine_geometry, build_cartesian, deform,
                   precompute_geometry)
from .cost import KernelCounter, scheme_cost, tck_cost_model

__all__ = [
    "AcousticOperator", "FluxParams", "StateVector", "hdg_flux", "LSRK45", "LSRK59", "RK4_CLASSIC",
    "SchemeConfig", "DeviceStepper", "ader_step", "advance", "compute_dt", "lsrk_step",
    "make_stepper", "rk_step", "state_norm", "tck_evaluate", "Material", "Mesh",
    "affine_geometry", "build_cartesian", "precompute_geometry", "CourantSearchError",
    "find_critical_courant", "exact_pressure_norm", "initial_state", "l2_pressure_error",
    "GeometryError", "deform", "KernelCounter", "scheme_cost", "tck_cost_model",
]
