"""The CPU oracle (oracle/) is pinned to golden vectors of the unmodified
reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest

import oracle
from oracle import quadrature as Q, stepping as OS
from helpers import Case, load, op_cases, rel, traj_cases

TOL = 1e-12


def test_tables_match_reference():
    z = load("tables")
    for k in range(1, 13):
        g, w = Q.gauss_rule(k + 1)
        assert np.abs(g - z[f"gauss_points_{k}"]).max() < 1e-15
        assert np.abs(w - z[f"gauss_weights_{k}"]).max() < 1e-15
        gl, glw = Q.gauss_lobatto_rule(k + 1)
        assert np.abs(gl - z[f"gl_points_{k}"]).max() < 1e-15
        assert np.abs(glw - z[f"gl_weights_{k}"]).max() < 1e-15
        B, Bi = Q.basis_change(k)
        scale = k * k
        assert np.abs(B - z[f"gl_to_g_{k}"]).max() < 1e-13
        assert np.abs(Bi - z[f"g_to_gl_{k}"]).max() < 1e-13 * scale
        assert np.abs(Q.gl_derivative_at_gauss(k) - z[f"d_gl_{k}"]).max() < 1e-13 * scale
        assert np.abs(Q.collocation_derivative(k) - z[f"d_co_{k}"]).max() < 1e-13 * scale
        for j in range(k + 1):
            assert np.abs(Q.projection_matrix(k, j) - z[f"proj_{k}_{j}"]).max() < 1e-13


@pytest.mark.parametrize("name", op_cases())
def test_operator_case(name):
    c = Case(name)
    z, op, u, dt = c.z, c.op, c.u, c.dt
    assert rel(op.apply_K(u), z["K_both"]) < TOL
    assert rel(op.apply_K(u, "cell"), z["K_cell"]) < TOL
    assert rel(op.apply_K(u, "face"), z["K_face"]) < TOL
    assert rel(op.apply_inverse_mass(u), z["Minv"]) < TOL
    assert rel(op.apply_mass(u), z["M"]) < TOL
    assert rel(op.rhs(u), z["rhs"]) < TOL
    vals = op.to_gauss_values(u)
    assert rel(vals, z["to_gauss"]) < TOL
    assert rel(op.from_gauss_weighted(vals), z["from_gauss_weighted"]) < TOL
    assert rel(op.apply_local_S(vals, c.k), z["localS_k"]) < TOL
    for q in c.reduced:
        assert rel(op.apply_local_S(z[f"localS_in_{q}"], q), z[f"localS_{q}"]) < TOL
        if q < c.k:
            assert rel(op.resize_values(vals, c.k, q), z[f"resize_down_{q}"]) < TOL
            assert rel(op.resize_values(z[f"localS_in_{q}"], q, c.k), z[f"resize_up_{q}"]) < TOL
    for pol in ("none", "every_second", "every_step", "every_third"):
        for sh in (0, 1):
            assert rel(OS.tck_evaluate(u, dt, op, pol, bool(sh)), z[f"tck_{pol}_{sh}"]) < TOL
    for var in ("ader", "ader_hdg"):
        for pol in ("none", "every_second"):
            assert rel(OS.ader_step(u, dt, op, var, pol), z[f"ader_{var}_{pol}"]) < TOL
    assert rel(OS.lsrk_step(u, dt, OS.LSRK45, op), z["lsrk45"]) < TOL
    assert rel(OS.lsrk_step(u, dt, OS.LSRK59, op), z["lsrk59"]) < TOL
    assert abs(OS.state_norm(op, u) - float(z["norm"])) < 1e-12 * float(z["norm"])


@pytest.mark.parametrize("name", traj_cases())
def test_trajectory_case(name):
    from paper_1805_03981_b200 import configs
    from paper_1805_03981_b200.configs import c3_mapping
    z = load("traj_" + name)
    prob = configs.config(str(z["config"]), scale=float(z["scale"]))
    assert np.array_equal(prob.state, z["u0"])
    m = prob.mesh
    om = oracle.OracleMesh(m.d, m.n_per_dim, m.vertices, m.elements, m.neighbors,
                           m.boundary_kind)
    k = prob.k
    if str(z["config"]) == "c3":
        base = oracle.build_cartesian(m.n_per_dim, 3, "periodic")
        geo = oracle.precompute_geometry(base, k, g=5, mapping=c3_mapping)
    else:
        geo = oracle.precompute_geometry(om, k)
    op = oracle.OracleOperator(om, geo, oracle.OracleMaterial(prob.material.c,
                                                              prob.material.rho))
    dt = float(z["dt"])
    assert abs(OS.compute_dt(float(z["courant"]), om, prob.material, k) - dt) < 1e-15 * dt
    scheme = str(z["scheme"])
    if scheme == "lsrk45":
        step = lambda u, h: OS.lsrk_step(u, h, OS.LSRK45, op)
    else:
        step = lambda u, h: OS.ader_step(u, h, op, scheme)
    u = OS.advance(z["u0"], dt, int(z["steps"]), step)
    assert rel(u, z["u_final"]) < 1e-10


@pytest.mark.parametrize("name", ["c2s8_lsrk45_100", "c3s8_ader_hdg_100"])
def test_long_trajectory_oracle(name):
    """100 steps (north_star's trajectory bar) of the oracle against the
    unmodified reference (tests/golden/make_golden_long.py); config 3 with
    the oracle's own degree-5 metric (~30 s each)."""
    from paper_1805_03981_b200 import configs
    from paper_1805_03981_b200.configs import c3_mapping
    z = load("long_" + name)
    cfg = str(z["config"])
    prob = configs.config(cfg, scale=float(z["scale"]))
    m = prob.mesh
    om = oracle.OracleMesh(m.d, m.n_per_dim, m.vertices, m.elements, m.neighbors,
                           m.boundary_kind)
    k = prob.k
    if cfg == "c3":
        base = oracle.build_cartesian(m.n_per_dim, 3, "periodic")
        geo = oracle.precompute_geometry(base, k, g=5, mapping=c3_mapping)
    else:
        geo = oracle.precompute_geometry(om, k)
    op = oracle.OracleOperator(om, geo, oracle.OracleMaterial(prob.material.c,
                                                              prob.material.rho))
    dt = float(z["dt"])
    scheme = str(z["scheme"])
    if scheme == "lsrk45":
        step = lambda u, h: OS.lsrk_step(u, h, OS.LSRK45, op)
    else:
        step = lambda u, h: OS.ader_step(u, h, op, scheme)
    u = OS.advance(prob.state, dt, int(z["steps"]), step)
    assert rel(u[z["ids"]], z["u_sample"]) < 1e-10
    assert abs(OS.state_norm(op, u) - float(z["norm"])) < 1e-10 * float(z["norm"])
