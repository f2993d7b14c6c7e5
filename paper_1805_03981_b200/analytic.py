"""Standing-mode initial state and L2 pressure error on the GPU.

Mirrors ``/root/reference/pkg/src/wavekernel/analytic.py``: the
pressure-release cavity mode (:1-12), ``exact_pressure_norm`` (:43-46),
``initial_state`` (:48-64) and ``l2_pressure_error`` (:67-93), same
signatures.  The fields are evaluated by the ``wk_mode_state`` /
``wk_l2_pressure_error`` kernels (csrc/wk_fields.cu) on the multilinear
vertex map of the mesh; states stay on the device (SURVEY.md §8f row 2:
convergence studies and stability guards without host round trips).
"""

from __future__ import annotations

import ctypes

import numpy as np

from ._lib import check, lib
from .operator import StateVector, _torch

__all__ = ["exact_pressure_norm", "initial_state", "l2_pressure_error"]


def exact_pressure_norm(t: float, m: int, c: float, d: int) -> float:
    """L2 norm of the mode pressure over the unit cube (analytic.py:43-46)."""
    omega = c * m * np.pi * np.sqrt(d)
    return abs(np.cos(omega * t)) * 0.5 ** (d / 2.0)


def _corners(mesh, device):
    torch = _torch()
    x = np.ascontiguousarray(mesh.vertices[mesh.elements], dtype=np.float64)  # (E, 2^d, d)
    return torch.from_numpy(x).to(device)


def _stream(device):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def initial_state(mesh, degree: int, material, m: int = 1, t: float = 0.0,
                  device: str = "cuda") -> StateVector:
    """The mode at the GL nodes of every element (analytic.py:48-64); uniform
    material assumed (material.c[0], material.rho[0]), like the reference."""
    torch = _torch()
    dev = torch.device(device)
    d, E, n = mesh.d, mesh.n_elements, degree + 1
    out = torch.empty((E, d + 1) + (n,) * d, dtype=torch.float64, device=dev)
    verts = _corners(mesh, dev)
    check(lib().wk_mode_state(d, int(degree), E, ctypes.c_void_p(verts.data_ptr()), int(m),
                              float(t), float(material.c[0]), float(material.rho[0]),
                              ctypes.c_void_p(out.data_ptr()), _stream(dev)))
    return StateVector(out, degree, d)


def l2_pressure_error(state: StateVector, mesh, material, t: float, m: int = 1,
                      n_extra: int = 2) -> float:
    """L2 distance of the pressure from the mode at time t on the
    (k+1+n_extra)-point Gauss rule (analytic.py:67-93)."""
    torch = _torch()
    data = state.data
    if isinstance(data, np.ndarray):
        data = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64)).cuda()
    data = data.contiguous()
    dev = data.device
    verts = _corners(mesh, dev)
    res = torch.empty(1, dtype=torch.float64, device=dev)
    check(lib().wk_l2_pressure_error(state.dim, state.degree, mesh.n_elements,
                                     ctypes.c_void_p(data.data_ptr()),
                                     ctypes.c_void_p(verts.data_ptr()), int(m), float(t),
                                     float(material.c[0]), float(material.rho[0]),
                                     int(n_extra), ctypes.c_void_p(res.data_ptr()),
                                     _stream(dev)))
    return float(np.sqrt(float(res.item())))
