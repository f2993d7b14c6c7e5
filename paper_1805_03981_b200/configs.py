"""The five BASELINE.json configurations, frozen.

BASELINE.json leaves some parameters open; they are frozen HERE, once, and
shared by the GPU path, the CPU oracle (tests / bench baseline) and the
golden-fixture generator:

* Fourier initial pressure (c2, c4, c5): p = sum_{j=1..8} a_j sin(2 pi kappa_j.x
  + phi_j), kappa_j in {1..4}^d (integer -> periodic), a_j ~ U(-1,1),
  phi_j ~ U(0, 2 pi), drawn from default_rng(seed) in the order kappa, a, phi;
  v = 0.  Seeds: c2 -> 2, c4 -> 4, c5 -> 5.
* Random materials (c3 seed 1, c5 seed 7): default_rng(seed), c drawn first
  then rho, both U(0.5, 2) per cell.
* c3 map: x -> x + 0.05 sin(2 pi x) sin(2 pi y) sin(2 pi z) (1,1,1) as a
  degree-5 isoparametric (GL-node) interpolant; the map vanishes on the cube
  boundary so the mesh stays periodic.  Pressure pulse exp(-|x-0.5|^2/0.01).
* c4 layers: x_2 < 1/2 -> (rho, c) = (1, 1), else (2, 0.5) (both Z = 1).
* Courant numbers: c1 0.2 (BASELINE), c2 0.2 (ADER-HDG 0.1), c3 0.1
  (LSRK45 0.2), c4 LSRK45 0.373 /
  ADER-HDG 0.163 (0.9 x the reference's own 3D k=7 critical values, SURVEY
  §8d), c5 LSRK45 0.2 / ADER-HDG 0.1.  Per-step throughput does not depend
  on Cr.
* ADER uses the reference defaults: variant ``ader_hdg``, reduction
  ``every_second`` (cli.py:76).  "ADER of order k+1".

All initial data are sampled at the GL nodes through the element map, like
the reference's initial_state (analytic.py:48-63).  ``scale`` shrinks the
per-axis element counts (parity tests run the same rules on small meshes).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import mesh as M
from . import rules


@dataclass
class Problem:
    name: str
    mesh: object
    geometry: object
    material: object
    state: np.ndarray          # (E, d+1, n, ..., n) GL coefficients
    k: int
    schemes: dict              # scheme -> (courant, steps)
    description: str

    @property
    def dofs(self) -> int:
        d = self.mesh.d
        return int(self.mesh.n_elements * (d + 1) * (self.k + 1) ** d)


def fourier_pressure(x: np.ndarray, seed: int, n_modes: int = 8) -> np.ndarray:
    d = x.shape[-1]
    rng = np.random.default_rng(seed)
    kappa = rng.integers(1, 5, size=(n_modes, d))
    amp = rng.uniform(-1.0, 1.0, size=n_modes)
    phase = rng.uniform(0.0, 2.0 * np.pi, size=n_modes)
    p = np.zeros(x.shape[:-1])
    for j in range(n_modes):
        p += amp[j] * np.sin(2.0 * np.pi * (x @ kappa[j]) + phase[j])
    return p


def random_material(n_elements: int, seed: int) -> M.Material:
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.5, 2.0, n_elements)
    rho = rng.uniform(0.5, 2.0, n_elements)
    return M.Material(c=c, rho=rho)


def c3_mapping(x: np.ndarray) -> np.ndarray:
    bump = 0.05 * np.prod(np.sin(2.0 * np.pi * x), axis=-1)
    return x + bump[..., None]


def _state(p: np.ndarray, d: int) -> np.ndarray:
    st = np.zeros((p.shape[0], d + 1) + p.shape[1:])
    st[:, d] = p
    return st


def _gl_coords(mesh, k, g=1, mapping=None):
    return M.map_points(mesh, rules.gl_points(k), g, mapping)


def config(name: str, scale: float = 1.0, geometry: str = "auto",
           state: bool = True) -> Problem:
    """Build config ``name`` in {c1..c5}; ``scale`` < 1 shrinks the mesh.

    ``geometry="device"``: config 3's curved metric is evaluated on the GPU
    (precompute_geometry(device="cuda")); "auto"/"host": on the host;
    "none": config 3 gets no geometry (callers that build their own, e.g.
    the CPU oracle arm of bench.py).  ``state=False`` skips the initial state
    (``Problem.state`` is then None; the ncu probe fills the device vector
    itself)."""
    def n(v):
        return max(2, int(round(v * scale)))

    def fourier(mesh, k, seed):
        return _state(fourier_pressure(_gl_coords(mesh, k), seed=seed), 3) if state else None

    if name == "c1":
        mesh = M.build_cartesian(n(16), 2, "periodic")
        k = 3
        mat = M.Material.uniform(mesh)
        u0 = None
        if state:
            x = _gl_coords(mesh, k)
            u0 = _state(np.sin(2 * np.pi * x[..., 0]) * np.sin(2 * np.pi * x[..., 1]), 2)
        geo = M.affine_geometry(mesh, k)
        return Problem(name, mesh, geo, mat, u0, k, {"lsrk45": (0.2, 10)},
                       "2D 16^2 periodic k=3 LSRK45 Cr 0.2 10 steps")
    if name == "c2":
        mesh = M.build_cartesian(n(32), 3, "periodic")
        k = 4
        mat = M.Material.uniform(mesh)
        geo = M.affine_geometry(mesh, k)
        return Problem(name, mesh, geo, mat, fourier(mesh, k, 2), k,
                       {"lsrk45": (0.2, 100), "ader_hdg": (0.1, 100)},
                       "3D 32^3 periodic k=4 LSRK45 100 steps")
    if name == "c3":
        base = M.build_cartesian(n(32), 3, "periodic")
        k = 5
        mesh = M.map_vertices(base, c3_mapping)
        geo = None
        if geometry != "none":
            geo = M.precompute_geometry(base, k, reduced_degrees=(3, 1), g=5,
                                        mapping=c3_mapping,
                                        device="cuda" if geometry == "device" else None)
        mat = random_material(mesh.n_elements, seed=1)
        u0 = None
        if state:
            x = _gl_coords(base, k, g=5, mapping=c3_mapping)
            u0 = _state(np.exp(-np.sum((x - 0.5) ** 2, axis=-1) / 0.01), 3)
        return Problem(name, mesh, geo, mat, u0, k, {"ader_hdg": (0.1, 50), "lsrk45": (0.2, 50)},
                       "3D 32^3 curved (degree-5 sin map) k=5 ADER-HDG order 6, 50 steps")
    if name == "c4":
        mesh = M.build_cartesian(n(48), 3, "periodic")
        k = 7
        xc = mesh.vertices[mesh.elements].mean(axis=1)
        upper = xc[:, 2] > 0.5
        mat = M.Material(c=np.where(upper, 0.5, 1.0), rho=np.where(upper, 2.0, 1.0))
        geo = M.affine_geometry(mesh, k)
        return Problem(name, mesh, geo, mat, fourier(mesh, k, 4), k,
                       {"ader_hdg": (0.163, 20), "lsrk45": (0.373, 20)},
                       "3D 48^3 periodic k=7 two-layer, ADER-HDG order 8 vs LSRK45, 20 steps")
    if name == "c5":
        nx, ny, nz = n(128), n(128), n(64)
        mesh = M.build_cartesian((nx, ny, nz), 3, "periodic")
        k = 4
        mat = random_material(mesh.n_elements, seed=7)
        geo = M.affine_geometry(mesh, k)
        return Problem(name, mesh, geo, mat, fourier(mesh, k, 5), k,
                       {"lsrk45": (0.2, 20), "ader_hdg": (0.1, 20)},
                       "3D 128x128x64 periodic k=4 random material, LSRK45 and ADER-HDG order 5")
    raise ValueError(f"unknown config {name!r}")
