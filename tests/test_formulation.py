"""CPU proof of the kernels' algebra (no GPU): the collapsed affine
formulation used by wk_affine.cuh / wk_stage.cuh and the GL-basis Taylor
loop of wk_tck.cuh reproduce the oracle (and hence the reference) to
round-off.  The numpy models below mirror the kernels step by step, with the
library's own natively computed tables.
"""

import numpy as np
import pytest

import oracle
from oracle import stepping as OS
from helpers import Case, rel

from paper_1805_03981_b200._lib import basis_table
from paper_1805_03981_b200 import mesh as PM

AFFINE_CASES = ["q2_periodic_k3", "q2_soft_sheared_k5", "h3_soft_k4", "h3_periodic_k7",
                "h3_periodic_k3_nostab", "h3_soft_sheared_k3"]


def _along(mat, arr, m):
    ax = arr.ndim - 1 - m
    return np.moveaxis(np.tensordot(arr, mat, axes=([ax], [1])), -1, ax)


def collapsed_minv_K(u, G, det, normal, fscale, ir, c2r, tau, nbr, k, d, stab=True):
    """M^{-1} K u as the affine kernels compute it."""
    A = basis_table("a_split", k)
    L = basis_table("lift", k)
    E = u.shape[0]
    bE = (slice(None),) + (None,) * d
    bF = (slice(None),) + (None,) * (d - 1)
    out = np.zeros_like(u)
    p = u[:, d]
    for m in range(d):
        dp = _along(A, p, m)
        w = sum(G[:, m, i][bE] * u[:, i] for i in range(d))
        for i in range(d):
            out[:, i] += (ir * G[:, m, i])[bE] * dp
        out[:, d] += c2r[bE] * _along(A, w, m)
    for m in range(d):
        ax = 2 + d - 1 - m
        for s in (0, 1):
            idx = [slice(None)] * (2 + d)
            idx[ax] = -1 if s else 0
            own = u[tuple(idx)]
            idx2 = list(idx)
            idx2[ax] = 0 if s else -1
            oth = u[tuple(idx2)][np.maximum(nbr[:, m, s], 0)].copy()
            wall = nbr[:, m, s] < 0
            oth[wall, :d] = own[wall, :d]
            oth[wall, d] = -own[wall, d]
            n = normal[:, m, s]
            vo = sum(n[:, i][bF] * own[:, i] for i in range(d))
            vx = sum(n[:, i][bF] * oth[:, i] for i in range(d))
            pv = 0.5 * ir[bF] * oth[:, d]
            pp = 0.5 * c2r[bF] * vx
            if stab:
                pv = pv + 0.5 * (ir / tau)[bF] * (vo - vx)
                pp = pp + 0.5 * (c2r * tau)[bF] * (own[:, d] - oth[:, d])
            F = np.concatenate([(pv * n[:, i][bF])[:, None] for i in range(d)]
                               + [pp[:, None]], axis=1) * fscale[:, m, s][(slice(None),) + (None,) * d]
            shape = [1] * d
            shape[d - 1 - m] = k + 1
            out += np.expand_dims(F, ax) * L[s].reshape(shape)[None, None]
    return out


def _affine_inputs(c):
    geo = PM.affine_geometry(c.mesh, c.k)
    ir = 1.0 / c.material.rho
    c2r = c.material.c ** 2 * c.material.rho
    tau = c.op.tau
    return geo, ir, c2r, tau


@pytest.mark.parametrize("name", AFFINE_CASES)
def test_collapsed_operator_equals_oracle(name):
    c = Case(name)
    geo, ir, c2r, tau = _affine_inputs(c)
    got = collapsed_minv_K(c.u, geo.G, geo.det, geo.normal, geo.fscale, ir, c2r, tau,
                           c.mesh.neighbors, c.k, c.d, c.stab)
    assert rel(got, -c.z["rhs"]) < 1e-13
    assert rel(got, c.op.apply_inverse_mass(c.op.apply_K(c.u))) < 1e-13


def gl_taylor(u, dt, G, ir, c2r, k, d, policy, shift):
    """The GL-basis Taylor loop program of wk_abi.cu::get_program, in numpy."""
    Dglco = PM.lagrange(basis_table("gl_points", k), basis_table("gl_points", k), True)
    B = basis_table("gl_to_g", k)
    bE = (slice(None),) + (None,) * d

    def S(x, dm):
        out = np.empty_like(x)
        p = x[:, d]
        dps = [_along(dm, p, m) for m in range(d)]
        for i in range(d):
            out[:, i] = ir[bE] * sum(G[:, m, i][bE] * dps[m] for m in range(d))
        out[:, d] = c2r[bE] * sum(_along(dm, sum(G[:, m, i][bE] * x[:, i] for i in range(d)), m)
                                  for m in range(d))
        return out

    def resize(x, a, b):
        if a == k:
            mat = basis_table("resize", k, b) @ B
        elif b == k:
            mat = PM.lagrange(basis_table("gauss_points", a), basis_table("gl_points", k))
        else:
            mat = basis_table("resize", a, b)
        for m in range(d):
            x = _along(mat, x, m)
        return x

    cur = u
    acc = {k: OS.taylor_weight(1 if shift else 0, dt) * cur}
    sched = OS.reduction_schedule(k, policy)
    deg = k
    for j in range(1, (max(k - 1, 0) if shift else k + 1) + 1):
        din, dout = sched[j - 1]
        if din == 0:
            break
        cur = S(cur, Dglco if deg == k else basis_table("d_co", deg))
        if dout != din:
            cur = resize(cur, deg, dout)
            deg = dout
        w = OS.taylor_weight(j + 1 if shift else j, dt)
        acc[deg] = acc[deg] + w * cur if deg in acc else w * cur
    for lo in sorted(acc):
        if lo == k:
            break
        hi = min(q for q in acc if q > lo)
        acc[hi] = acc[hi] + resize(acc[lo], lo, hi)
    return acc[k]          # GL coefficients = M^{-1} T


@pytest.mark.parametrize("name", ["q2_periodic_k3", "h3_soft_k4", "h3_periodic_k7",
                                  "h3_soft_sheared_k3"])
@pytest.mark.parametrize("policy", ["none", "every_second", "every_step", "every_third"])
@pytest.mark.parametrize("shift", [False, True])
def test_gl_taylor_loop_equals_oracle(name, policy, shift):
    c = Case(name)
    geo, ir, c2r, _ = _affine_inputs(c)
    got = gl_taylor(c.u, c.dt, geo.G, ir, c2r, c.k, c.d, policy, shift)
    ref = c.op.apply_inverse_mass(c.z[f"tck_{policy}_{int(shift)}"])
    assert rel(got, ref) < 1e-12
