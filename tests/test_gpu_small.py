"""Whole-run LSRK in one thread-block-cluster launch (csrc/wk_small.cuh,
wk_lsrk_run) for small Cartesian meshes -- BASELINE config 1.

The cluster kernel keeps the state in the CTAs' shared memories, reads the
neighbours' faces through distributed shared memory and synchronises the
stages with cluster barriers; its arithmetic mirrors the stage kernel's
operation order, so K steps must be BITWISE equal to K x S stage launches,
and config 1 in full must match the unmodified reference's trajectory
(tests/golden/traj_c1_lsrk45_10.npz)."""

import ctypes

import numpy as np
import pytest
import torch

from helpers import load, rel

pytestmark = pytest.mark.gpu


def _stage_path(op, u, dt, scheme, steps):
    from paper_1805_03981_b200._lib import check, lib
    cur, nxt, r = u.clone(), torch.empty_like(u), torch.empty_like(u)
    for _ in range(steps):
        for a, b in zip(scheme.a, scheme.b):
            check(lib().wk_lsrk_stage(op._ctx, op._ptr(cur), op._ptr(nxt), op._ptr(r), float(a),
                                      float(b), float(dt), op.stream))
            cur, nxt = nxt, cur
    return cur


@pytest.mark.parametrize("d,n,k,bk", [(2, 16, 3, "periodic"), (2, 12, 5, "sound_soft"),
                                      (3, 4, 4, "periodic"), (2, 40, 2, "periodic"),
                                      (3, 3, 3, "sound_soft"), (2, 5, 8, "periodic")])
@pytest.mark.parametrize("scheme", ["lsrk45", "lsrk59"])
def test_cluster_run_bitwise_equals_stage_launches(d, n, k, bk, scheme, cuda):
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import mesh as M
    from paper_1805_03981_b200._lib import check, lib
    rng = np.random.default_rng(d * 100 + n + k)
    mesh = M.build_cartesian(n, d, bk)
    E = mesh.n_elements
    mat = M.Material(c=rng.uniform(0.5, 2, E), rho=rng.uniform(0.5, 2, E))
    op = W.AcousticOperator(mesh, M.affine_geometry(mesh, k), mat)
    assert op.small_run
    sch = W.LSRK45 if scheme == "lsrk45" else W.LSRK59
    u0 = torch.from_numpy(rng.standard_normal((E, d + 1) + (k + 1,) * d)).to(cuda)
    dt = W.compute_dt(0.2, mesh, mat, k)
    ref = _stage_path(op, u0, dt, sch, 7)
    got = u0.clone()
    st = sch.stages
    check(lib().wk_lsrk_run(op._ctx, op._ptr(got), op._ptr(got), st,
                            (ctypes.c_double * st)(*sch.a), (ctypes.c_double * st)(*sch.b),
                            float(dt), 7, op.stream))
    torch.cuda.synchronize()
    assert torch.equal(got, ref)


def test_config1_full_trajectory(cuda):
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import configs
    z = load("traj_c1_lsrk45_10")
    prob = configs.config("c1")
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    assert op.small_run
    stepper = W.make_stepper(W.SchemeConfig(scheme="lsrk45"), op)
    out = W.advance(W.StateVector(torch.from_numpy(z["u0"]).to(cuda), prob.k, 2),
                    float(z["dt"]), int(z["steps"]), stepper).data.cpu().numpy()
    assert rel(out, z["u_final"]) < 1e-10


def test_large_mesh_not_eligible(cuda):
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import configs
    prob = configs.config("c2", scale=0.5)          # 16^3 k=4: 16 MB of state
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    assert not op.small_run
