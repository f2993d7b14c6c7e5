"""Every supported degree (k = 1..8, the whole compiled instantiation range)
in 2-D and 3-D, straight (per-element affine metric) and deformed (per-point
metric) cells, periodic and sound-soft boundaries, random per-cell materials:
rhs, one LSRK45 step and one step of each ADER variant against the oracle
(tolerance: north_star's 1e-12 relative L2 per operator application/step).
The reference golden cases pin k = 2..7; this sweep adds the range ends
(k = 1: an empty shifted Taylor loop; k = 8: the largest tiles)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import stepping as OS
from helpers import rel

pytestmark = pytest.mark.gpu

CASES = [(d, k, bk, deformed)
         for d in (2, 3) for k in range(1, 9)
         for bk, deformed in (("periodic", False), ("sound_soft", True))
         if not (deformed and k == 8)]     # curved kernels support k <= 7


@pytest.mark.parametrize("d,k,bk,deformed", CASES)
def test_degree_sweep(d, k, bk, deformed, cuda):
    import torch
    import paper_1805_03981_b200 as W
    n = 3 if d == 3 else 4
    mesh = W.build_cartesian(n, d, bk)
    if deformed:
        mesh = W.deform(mesh, 0.05)
    rng = np.random.default_rng(100 * d + k)
    c, rho = rng.uniform(0.5, 2, mesh.n_elements), rng.uniform(0.5, 2, mesh.n_elements)
    mat = W.Material(c=c, rho=rho)
    reduced = tuple(sorted(set(W.stepping.reduction_degrees(k, "every_second"))
                           | set(W.stepping.reduction_degrees(k, "none")), reverse=True))
    om = oracle.OracleMesh(d, mesh.n_per_dim, mesh.vertices, mesh.elements, mesh.neighbors, bk)
    ogeo = oracle.precompute_geometry(om, k, reduced)
    oop = oracle.OracleOperator(om, ogeo, oracle.OracleMaterial(c, rho))
    geo = W.precompute_geometry(mesh, k, reduced_degrees=reduced) if deformed \
        else W.affine_geometry(mesh, k)
    op = W.AcousticOperator(mesh, geo, mat)
    u = rng.standard_normal((mesh.n_elements, d + 1) + (k + 1,) * d)
    st = W.StateVector(torch.from_numpy(u).to(cuda), k, d)
    dt = 0.5 * W.compute_dt(0.1, mesh, mat, k)
    assert rel(op.rhs(st).data.cpu().numpy(), oop.rhs(u)) < 1e-12
    got = W.lsrk_step(st, dt, W.LSRK45, op).data.cpu().numpy()
    assert rel(got, OS.lsrk_step(u, dt, OS.LSRK45, oop)) < 1e-12
    for variant in ("ader_hdg", "ader"):
        got = W.ader_step(st, dt, op, variant, "every_second").data.cpu().numpy()
        assert rel(got, OS.ader_step(u, dt, oop, variant, "every_second")) < 1e-12, variant
