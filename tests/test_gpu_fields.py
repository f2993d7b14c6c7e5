"""Fields around the time loop on the GPU against
the reference's own outputs (tests/golden/make_golden_fields.py ran the
unmodified reference): the mode initial state, the L2 pressure error, the
fused state norm and the critical Courant search."""

import numpy as np
import pytest
import torch

from helpers import load, rel

pytestmark = pytest.mark.gpu

Z = load("fields")
MESHES = sorted({k.split("/")[0] for k in Z if not k.startswith("courant")})
COURANT = sorted({k.split("/")[1] for k in Z if k.startswith("courant/") and k.count("/") == 1})


def _mesh(name):
    from paper_1805_03981_b200.mesh import Mesh
    d, n, k, m, per = (int(v) for v in Z[f"{name}/meta"])
    mesh = Mesh(d, (n,) * d, Z[f"{name}/vertices"], Z[f"{name}/elements"],
                Z[f"{name}/neighbors"], "periodic" if per else "sound_soft")
    return mesh, k, m, float(Z[f"{name}/t"])


@pytest.mark.parametrize("name", MESHES)
def test_initial_state_matches_reference(name, cuda):
    import paper_1805_03981_b200 as W
    mesh, k, m, t = _mesh(name)
    mat = W.Material.uniform(mesh)
    s0 = W.initial_state(mesh, k, mat, m=m)
    assert s0.data.is_cuda and s0.degree == k and s0.dim == mesh.d
    assert rel(s0.data.cpu().numpy(), Z[f"{name}/init0"]) < 1e-13
    st = W.initial_state(mesh, k, mat, m=m, t=t)
    assert rel(st.data.cpu().numpy(), Z[f"{name}/init_t"]) < 1e-13


@pytest.mark.parametrize("name", MESHES)
def test_l2_error_and_norm_match_reference(name, cuda):
    import paper_1805_03981_b200 as W
    mesh, k, m, t = _mesh(name)
    mat = W.Material.uniform(mesh)
    pert = W.StateVector(torch.from_numpy(Z[f"{name}/pert"]).cuda(), k, mesh.d)
    err = W.l2_pressure_error(pert, mesh, mat, t, m=m)
    assert err == pytest.approx(float(Z[f"{name}/l2_pert"]), rel=1e-12)
    # interpolation error of the exact mode: tiny, compared absolutely
    exact = W.initial_state(mesh, k, mat, m=m, t=t)
    e0 = W.l2_pressure_error(exact, mesh, mat, t, m=m)
    assert abs(e0 - float(Z[f"{name}/l2_exact"])) < 1e-12 * max(1.0, float(Z[f"{name}/l2_pert"]))
    # host (numpy) state through the same kernels
    assert W.l2_pressure_error(W.StateVector(Z[f"{name}/pert"], k, mesh.d), mesh, mat, t,
                               m=m) == pytest.approx(err, rel=1e-15)
    geo = W.precompute_geometry(mesh, k, device="cuda")
    op = W.AcousticOperator(mesh, geo, mat)
    nrm = W.state_norm(op, pert)
    assert nrm == pytest.approx(float(Z[f"{name}/norm_pert"]), rel=1e-12)
    assert W.state_norm(op, W.StateVector(Z[f"{name}/pert"], k, mesh.d)) == pytest.approx(
        nrm, rel=1e-15)


@pytest.mark.parametrize("name", COURANT)
def test_critical_courant_matches_reference(name, cuda):
    import paper_1805_03981_b200 as W
    n, k, width, n_steps = Z[f"courant/{name}/args"]
    scheme = name.rsplit("_k", 1)[0]
    mesh = W.build_cartesian(int(n), 2, "sound_soft")
    cr = W.find_critical_courant(W.SchemeConfig(scheme=scheme), mesh, int(k),
                                 width=float(width), n_steps=int(n_steps))
    assert cr == pytest.approx(float(Z[f"courant/{name}"]), abs=1e-12)


def test_courant_search_errors(cuda):
    """tests/test_stepping.py:366-372"""
    import paper_1805_03981_b200 as W
    mesh = W.build_cartesian(4, 2, "sound_soft")
    cfg = W.SchemeConfig(scheme="lsrk45")
    with pytest.raises(W.CourantSearchError):
        W.find_critical_courant(cfg, mesh, 1, lo=0.01, hi=0.05, n_steps=200)
    with pytest.raises(W.CourantSearchError):
        W.find_critical_courant(cfg, mesh, 1, lo=1.5, hi=2.0, n_steps=200)


def test_exact_pressure_norm():
    import paper_1805_03981_b200 as W
    assert W.exact_pressure_norm(0.0, 1, 1.0, 2) == pytest.approx(0.5)
    assert W.exact_pressure_norm(0.0, 2, 1.0, 3) == pytest.approx(0.5 ** 1.5)
