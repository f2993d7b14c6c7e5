"""Curved geometry evaluated on the device (wk_curved_metric, SURVEY.md §8f
row 1) against the oracle's GeometryCache arrays (reference mesh.py:245-334),
and the operator / a config-3 trajectory run on it against the golden
vectors."""

import numpy as np
import pytest
import torch

import oracle
from helpers import Case, load, op_cases, rel

pytestmark = pytest.mark.gpu


def _device_geometry(c):
    from paper_1805_03981_b200 import mesh as M
    from paper_1805_03981_b200.configs import c3_mapping
    if c.curved:
        base = oracle.build_cartesian(c.mesh.n_per_dim, c.d, c.mesh.boundary_kind)
        return M.precompute_geometry(base, c.k, c.reduced, g=5, mapping=c3_mapping,
                                     device="cuda")
    return M.precompute_geometry(c.mesh, c.k, c.reduced, device="cuda")


def _maxrel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())


@pytest.mark.parametrize("name", op_cases())
def test_device_geometry_matches_oracle(name, cuda):
    """Independent builders (device double-double vs the oracle's long
    double, different GL/Gauss point routines) agree to a few ulp: the metric
    of the interpolated map is reproducible, not builder-dependent."""
    c = Case(name)
    geo = _device_geometry(c)
    ref = c.geometry
    for q, v in ref.vol.items():
        assert _maxrel(geo.vol[q].inv_jac.cpu().numpy(), v.inv_jac) < 2e-15, q
        assert _maxrel(geo.vol[q].jxw.cpu().numpy(), v.jxw) < 4e-15, q
    for f, v in ref.face.items():
        assert _maxrel(geo.face[f].normal.cpu().numpy(), v.normal) < 2e-15, f
        assert _maxrel(geo.face[f].jxw.cpu().numpy(), v.jxw) < 4e-15, f
    assert np.array_equal(np.asarray(geo.cartesian_flag), np.asarray(ref.cartesian_flag))
    assert geo.h_min == pytest.approx(ref.h_min, rel=1e-14)


@pytest.mark.parametrize("name", [n for n in op_cases() if "curved" in n or "deformed" in n])
def test_device_geometry_matches_host_builder(name, cuda):
    """Device (double-double) and host (long double) product builders: same
    tables and weights, so the rounded results agree to 1 ulp."""
    from paper_1805_03981_b200 import mesh as M
    from paper_1805_03981_b200.configs import c3_mapping
    c = Case(name)
    dev = _device_geometry(c)
    if c.curved:
        base = M.build_cartesian(c.mesh.n_per_dim, c.d, c.mesh.boundary_kind)
        host = M.precompute_geometry(base, c.k, c.reduced, g=5, mapping=c3_mapping)
    else:
        host = M.precompute_geometry(c.mesh, c.k, c.reduced)
    for q, v in host.vol.items():
        assert _maxrel(dev.vol[q].inv_jac.cpu().numpy(), v.inv_jac) < 5e-16, q
        assert _maxrel(dev.vol[q].jxw.cpu().numpy(), v.jxw) < 5e-16, q
    for f, v in host.face.items():
        assert _maxrel(dev.face[f].normal.cpu().numpy(), v.normal) < 5e-16, f
        assert _maxrel(dev.face[f].jxw.cpu().numpy(), v.jxw) < 5e-16, f


@pytest.mark.parametrize("name", [n for n in op_cases() if "curved" in n or "deformed" in n])
def test_operator_on_device_geometry(name, cuda):
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200.operator import FluxParams
    c = Case(name)
    op = W.AcousticOperator(c.mesh, _device_geometry(c), c.material,
                            flux=FluxParams(tau=c.tau, stabilization=c.stab))
    assert op.geometry_mode == "curved"
    st = W.StateVector(torch.from_numpy(c.u).cuda(), c.k, c.d)
    assert rel(op.apply_K(st).data.cpu().numpy(), c.z["K_both"]) < 1e-12
    assert rel(op.rhs(st).data.cpu().numpy(), c.z["rhs"]) < 1e-12
    got = W.ader_step(st, c.dt, op, "ader_hdg", "every_second").data.cpu().numpy()
    assert rel(got, c.z["ader_ader_hdg_every_second"]) < 1e-12


def test_c3_trajectory_device_geometry(cuda):
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import configs
    z = load("traj_c3s_ader_hdg_10")
    prob = configs.config("c3", scale=float(z["scale"]), geometry="device")
    assert prob.geometry.vol[prob.k].inv_jac.is_cuda
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    stepper = W.make_stepper(W.SchemeConfig(scheme=str(z["scheme"])), op)
    st = W.StateVector(torch.from_numpy(z["u0"]).cuda(), prob.k, prob.mesh.d)
    out = W.advance(st, float(z["dt"]), int(z["steps"]), stepper).data.cpu().numpy()
    assert rel(out, z["u_final"]) < 1e-10
