"""The patch method behind the full-size GPU parity tests
(tests/test_gpu_fullsize.py), checked on the CPU: the oracle run on a patch
of face distance r around sampled elements reproduces the full-mesh oracle
at those elements exactly — r = 1 for one operator application, 2 for an
ADER-HDG step, 5 for an LSRK45 step (5 operator applications)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import stepping as OS
from helpers import patch, patch_operator


def _mesh(curved):
    m = oracle.build_cartesian((5, 4, 6), 3, "periodic")
    return m


@pytest.mark.parametrize("curved", [False, True])
def test_patch_reproduces_full_mesh(curved):
    m, k = _mesh(curved), 3
    rng = np.random.default_rng(3)
    c = rng.uniform(0.5, 2, m.n_elements)
    rho = rng.uniform(0.5, 2, m.n_elements)
    kw = {}
    if curved:
        from paper_1805_03981_b200.configs import c3_mapping
        kw = dict(g=3, mapping=c3_mapping)
    geo = oracle.precompute_geometry(m, k, (1,), **kw)
    op = oracle.OracleOperator(m, geo, oracle.OracleMaterial(c, rho))
    u = rng.standard_normal((m.n_elements, 4) + (k + 1,) * 3)
    cent = [0, 17, m.n_elements - 1]
    for r, fn in ((1, lambda o, x: o.rhs(x)),
                  (2, lambda o, x: OS.ader_step(x, 1e-2, o, "ader_hdg")),
                  (5, lambda o, x: OS.lsrk_step(x, 1e-2, OS.LSRK45, o))):
        ids, loc, ci = patch(m, cent, r)
        po = patch_operator(m, ids, loc, k, c, rho, (1,), **kw)
        np.testing.assert_array_equal(fn(po, u[ids])[ci], fn(op, u)[cent])


def test_patch_sound_soft_walls_kept():
    m = oracle.build_cartesian(3, 3, "sound_soft")
    ids, loc, ci = patch(m, [0], 1)
    assert (loc[ci[0]] == -1).sum() == 3          # the corner element's three walls
