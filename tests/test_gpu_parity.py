"""GPU parity: every operator and stepper through the C ABI against the CPU
oracle (pinned to the reference) and the reference's golden vectors.

Tolerance (BASELINE north_star): 1e-12 relative L2 per operator application,
1e-10 after multi-step trajectories.
"""

import numpy as np
import pytest
import torch

import oracle
from oracle import stepping as OS
from helpers import Case, load, op_cases, rel, traj_cases

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module", params=op_cases())
def case(request, cuda):
    c = Case(request.param)
    c.gop = c.gpu_operator()
    return c


def test_apply_K_parts(case):
    import paper_1805_03981_b200 as W
    st = W.StateVector(_dev(case.u), case.k, case.d)
    for parts, key in (("both", "K_both"), ("cell", "K_cell"), ("face", "K_face")):
        got = case.gop.apply_K(st, parts).data.cpu().numpy()
        assert rel(got, case.z[key]) < TOL, parts
        assert rel(got, case.op.apply_K(case.u, parts)) < TOL, parts


def test_mass_rhs(case):
    import paper_1805_03981_b200 as W
    st = W.StateVector(case.u, case.k, case.d)      # numpy in -> numpy out
    assert rel(case.gop.apply_inverse_mass(st).data, case.z["Minv"]) < TOL
    assert rel(case.gop.apply_mass(st).data, case.z["M"]) < TOL
    assert rel(case.gop.rhs(st).data, case.z["rhs"]) < TOL
    assert rel(case.gop.apply_minv_K(st).data, -case.z["rhs"]) < TOL


def test_local_operators(case):
    z, g = case.z, case.gop
    vals = g.to_gauss_values(case.u)
    assert rel(vals, z["to_gauss"]) < TOL
    assert rel(g.from_gauss_weighted(z["to_gauss"]), z["from_gauss_weighted"]) < TOL
    assert rel(g.apply_local_S(z["to_gauss"], case.k), z["localS_k"]) < TOL
    for q in case.reduced:
        assert rel(g.apply_local_S(z[f"localS_in_{q}"], q), z[f"localS_{q}"]) < TOL
        if q < case.k:
            assert rel(g.resize_values(z["to_gauss"], case.k, q), z[f"resize_down_{q}"]) < TOL
            assert rel(g.resize_values(z[f"localS_in_{q}"], q, case.k), z[f"resize_up_{q}"]) < TOL


def test_tck(case):
    import paper_1805_03981_b200 as W
    st = W.StateVector(_dev(case.u), case.k, case.d)
    for pol in ("none", "every_second", "every_step", "every_third"):
        for sh in (0, 1):
            got = W.tck_evaluate(st, case.dt, case.gop, pol, bool(sh)).data.cpu().numpy()
            assert rel(got, case.z[f"tck_{pol}_{sh}"]) < TOL, (pol, sh)


def test_ader_step(case):
    import paper_1805_03981_b200 as W
    st = W.StateVector(_dev(case.u), case.k, case.d)
    for var in ("ader", "ader_hdg"):
        for pol in ("none", "every_second"):
            got = W.ader_step(st, case.dt, case.gop, var, pol).data.cpu().numpy()
            assert rel(got, case.z[f"ader_{var}_{pol}"]) < TOL, (var, pol)


def test_lsrk_steps(case):
    import paper_1805_03981_b200 as W
    st = W.StateVector(_dev(case.u), case.k, case.d)
    assert rel(W.lsrk_step(st, case.dt, W.LSRK45, case.gop).data.cpu().numpy(),
               case.z["lsrk45"]) < TOL
    assert rel(W.lsrk_step(st, case.dt, W.LSRK59, case.gop).data.cpu().numpy(),
               case.z["lsrk59"]) < TOL
    assert rel(W.rk_step(st, case.dt, W.RK4_CLASSIC, case.gop).data.cpu().numpy(),
               case.z["rk4"]) < TOL
    assert abs(W.state_norm(case.gop, st) - float(case.z["norm"])) < 1e-12 * float(case.z["norm"])


def test_composed_path_matches_fused(case):
    """A duck-typed proxy forces the reference's composed call sequence
    (like tests/test_stepping.py:305-328); it must agree with the fused kernels."""
    import paper_1805_03981_b200 as W

    class Proxy:
        def __init__(self, inner):
            self._inner = inner
            self.calls = {}

        def __getattr__(self, name):
            attr = getattr(self._inner, name)
            if callable(attr):
                def wrapped(*a, **kw):
                    self.calls[name] = self.calls.get(name, 0) + 1
                    return attr(*a, **kw)
                return wrapped
            return attr

    st = W.StateVector(_dev(case.u), case.k, case.d)
    p = Proxy(case.gop)
    got = W.ader_step(st, case.dt, p, "ader_hdg").data.cpu().numpy()
    assert rel(got, case.z["ader_ader_hdg_every_second"]) < TOL
    assert p.calls["apply_K"] == 2 and p.calls["apply_inverse_mass"] == 3
    got = W.tck_evaluate(st, case.dt, p, "every_second", True).data.cpu().numpy()
    assert rel(got, case.z["tck_every_second_1"]) < TOL
    got = W.lsrk_step(st, case.dt, W.LSRK45, p).data.cpu().numpy()
    assert rel(got, case.z["lsrk45"]) < TOL
    assert p.calls["rhs"] == 5


@pytest.mark.parametrize("name", traj_cases())
def test_trajectory(name, cuda):
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import configs
    z = load("traj_" + name)
    prob = configs.config(str(z["config"]), scale=float(z["scale"]))
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    scheme = str(z["scheme"])
    stepper = W.make_stepper(W.SchemeConfig(scheme=scheme), op)
    st = W.StateVector(_dev(z["u0"]), prob.k, prob.mesh.d)
    out = W.advance(st, float(z["dt"]), int(z["steps"]), stepper).data.cpu().numpy()
    assert rel(out, z["u_final"]) < 1e-10


def test_errors_mirror_reference(cuda):
    import paper_1805_03981_b200 as W
    c = Case("q2_periodic_k3")
    g = c.gpu_operator()
    st = W.StateVector(_dev(c.u), c.k, c.d, basis="g")
    with pytest.raises(ValueError):
        g.apply_K(st)
    with pytest.raises(ValueError):
        g.apply_K(W.StateVector(_dev(c.u[:, :, :2]), c.k, c.d))
    with pytest.raises(ValueError):
        W.AcousticOperator(c.mesh, c.geometry, c.material, flux=W.FluxParams(tau=-1.0))
