"""north_star's trajectory bar: 1e-10 after 100 time steps, against the
UNMODIFIED reference (tests/golden/make_golden_long.py: 100 steps of
``wavekernel.stepping.advance``, stepping.py:305-308).

Cases: 8^3 versions of the config 2, 3 (curved, ADER-HDG) and 4 (both
schemes) rules, a 16x16x8 version of the config 5 rules (both schemes), and
config 2 at its full BASELINE size (32^3, k=4, 16.4 M DoF).  Each runs through
the production path: ``make_stepper`` -> ``DeviceStepper`` (fused kernels,
CUDA-graph replay); config 3 on the DEVICE-built curved metric, i.e. exactly
the geometry the bench times, while the reference ran on the oracle-built
metric (independent builders, agreeing to ~1 ulp, tests/test_gpu_geometry.py).

The fixtures hold the final state at seeded sampled elements plus full-state
checksums (per-component sum of squares and the mass norm); both are compared
at 1e-10 relative."""

from __future__ import annotations

import glob
import os

import numpy as np
import pytest

from helpers import GOLDEN, load, rel

pytestmark = pytest.mark.gpu

CASES = sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(GOLDEN, "long_*.npz")))


@pytest.mark.parametrize("name", CASES)
def test_long_trajectory(name, cuda):
    import torch
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import configs
    z = load("long_" + name)
    cfg = str(z["config"])
    prob = configs.config(cfg, scale=float(z["scale"]),
                          geometry="device" if cfg == "c3" else "auto")
    assert prob.mesh.n_elements == int(z["n_elements"])
    assert abs(np.sum(prob.state ** 2) - float(z["u0_sumsq"])) <= 1e-14 * float(z["u0_sumsq"])
    op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
    scheme = str(z["scheme"])
    dt = W.compute_dt(float(z["courant"]), prob.mesh, prob.material, prob.k)
    assert abs(dt - float(z["dt"])) <= 1e-15 * dt
    stepper = W.make_stepper(W.SchemeConfig(scheme=scheme, courant=float(z["courant"])), op)
    st = W.StateVector(torch.from_numpy(prob.state).to(cuda), prob.k, prob.mesh.d)
    out = W.advance(st, dt, int(z["steps"]), stepper)
    ids = torch.as_tensor(z["ids"], device=cuda)
    got = out.data.index_select(0, ids).cpu().numpy()
    assert rel(got, z["u_sample"]) <= 1e-10
    u = out.data
    sumsq = (u * u).sum(dim=tuple(i for i in range(u.dim()) if i != 1)).cpu().numpy()
    assert np.all(np.abs(sumsq - z["sumsq"]) <= 1e-10 * np.abs(z["sumsq"]).max())
    norm = W.state_norm(op, out)
    assert abs(norm - float(z["norm"])) <= 1e-10 * float(z["norm"])
