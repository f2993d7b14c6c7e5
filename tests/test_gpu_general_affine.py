"""General affine meshes (sheared, graded = multi-class) at sizes where every
persistent CTA processes several tiles, against the oracle on element patches
(reference operator.py:149-258, stepping.py:179-285).

Round 1's "fault above ~2k elements" on these meshes was the stage kernel
(wk_stage.cuh, LSRK / rhs / ADER kernel B of general affine meshes): its second
shared-memory stage and its r tile started 8 bytes off a 16-byte boundary
whenever the element tile or the 2-D geometry record times an odd number of
elements per block was odd, and 16-byte cp.async into it faulted once a CTA
reached its second tile.  These cases cover odd n in 2-D (EPB odd) and both
geometry classes, one ADER-HDG step (composed kernel A + stage kernel B) and
one LSRK45 step, at 1e-12."""

from __future__ import annotations

import numpy as np
import pytest

from helpers import patch, patch_operator, rel
from oracle import stepping as OS

pytestmark = pytest.mark.gpu

CASES = [(2, 64, 5, "shear"), (2, 48, 3, "graded"), (2, 40, 8, "shear"), (2, 36, 4, "graded_shear"),
         (3, 16, 3, "shear"), (3, 14, 4, "graded"), (3, 10, 6, "shear"), (3, 8, 7, "graded_shear")]


def _mesh(d, n, kind, rng):
    from paper_1805_03981_b200 import mesh as M
    m = M.build_cartesian(n, d, "periodic")
    v = m.vertices.copy()
    if "graded" in kind:
        for j in range(d):
            g = np.cumsum(rng.uniform(0.5, 1.5, n + 1))
            g = (g - g[0]) / (g[-1] - g[0])
            v[:, j] = g[np.rint(v[:, j] * n).astype(int)]
    if "shear" in kind:
        v = v @ (np.eye(d) + 0.2 * rng.standard_normal((d, d))).T
    return M.Mesh(m.d, m.n_per_dim, v, m.elements, m.neighbors, m.boundary_kind)


@pytest.mark.parametrize("d,n,k,kind", CASES)
def test_general_affine_steps_match_oracle(d, n, k, kind, cuda):
    import torch
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import mesh as M
    rng = np.random.default_rng(100 * d + n + k)
    mesh = _mesh(d, n, kind, rng)
    E = mesh.n_elements
    mat = M.Material(c=rng.uniform(0.5, 2, E), rho=rng.uniform(0.5, 2, E))
    op = W.AcousticOperator(mesh, M.affine_geometry(mesh, k), mat)
    if "graded" in kind:
        assert op.n_geometry_classes > 1
    u0 = rng.standard_normal((E, d + 1) + (k + 1,) * d)
    dt = 0.1 * W.compute_dt(0.2, mesh, mat, k)
    x = torch.from_numpy(u0).to(cuda)
    got_a = W.ader_step(W.StateVector(x, k, d), dt, op, "ader_hdg", "every_second").data
    got_l = W.lsrk_step(W.StateVector(x, k, d), dt, W.LSRK45, op).data
    torch.cuda.synchronize()
    centers = sorted({0, E - 1, *rng.integers(0, E, 3).tolist()})
    idx = torch.as_tensor(centers, device=cuda)
    got_a = got_a.index_select(0, idx).cpu().numpy()
    got_l = got_l.index_select(0, idx).cpu().numpy()
    reduced = W.stepping.reduction_degrees(k, "every_second")
    ref_a, ref_l = [], []
    for c in centers:
        ids, loc, ci = patch(mesh, [c], 2)
        po = patch_operator(mesh, ids, loc, k, mat.c, mat.rho, reduced)
        ref_a.append(OS.ader_step(u0[ids], dt, po, "ader_hdg")[ci[0]])
        ids, loc, ci = patch(mesh, [c], 5)
        po = patch_operator(mesh, ids, loc, k, mat.c, mat.rho)
        ref_l.append(OS.lsrk_step(u0[ids], dt, OS.LSRK45, po)[ci[0]])
    base = u0[centers]
    for got, ref in ((got_a, np.stack(ref_a)), (got_l, np.stack(ref_l))):
        assert rel(got, ref) <= 1e-12
        assert rel(got - base, ref - base) <= 1e-10
