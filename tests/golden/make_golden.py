"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container (the reference is importable only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Each operator case stores its inputs (mesh
arrays, material, flux, seeded random state) and the reference's outputs
(apply_K both/cell/face, apply_inverse_mass, apply_mass, rhs, apply_local_S,
tck_evaluate, ader_step, lsrk_step).  Trajectory cases store the input state
built by ``paper_1805_03981_b200.configs`` (same frozen rules as the bench)
and the reference's state after n steps.  Curved cases feed the reference's
own ``AcousticOperator`` a geometry built by ``oracle.precompute_geometry``
(the reference mesh code cannot build degree-5 maps).
"""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import wavekernel  # noqa: E402
from wavekernel import mesh as RM, operator as RO, quadrature as RQ, stepping as RS  # noqa: E402
from wavekernel.operator import FluxParams, StateVector  # noqa: E402

import oracle  # noqa: E402
from paper_1805_03981_b200 import configs  # noqa: E402


def tables():
    out = {}
    for k in range(1, 13):
        n = k + 1
        g, gl = RQ.gauss_rule(n), RQ.gauss_lobatto_rule(n)
        b, bi = RQ.basis_change_matrices(k)
        out[f"gauss_points_{k}"] = g.points
        out[f"gauss_weights_{k}"] = g.weights
        out[f"gl_points_{k}"] = gl.points
        out[f"gl_weights_{k}"] = gl.weights
        out[f"gl_to_g_{k}"] = b.matrix
        out[f"g_to_gl_{k}"] = bi.matrix
        out[f"d_gl_{k}"] = RQ.lagrange_matrix(gl.points, g.points, "derivative").matrix
        out[f"d_co_{k}"] = RQ.lagrange_matrix(g.points, g.points, "derivative").matrix
        for j in range(k + 1):
            out[f"proj_{k}_{j}"] = RQ.projection_matrix(k, j).matrix
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)


def _oracle_geometry(rmesh, k, g, mapping, reduced):
    om = oracle.OracleMesh(rmesh.d, rmesh.n_per_dim, rmesh.vertices, rmesh.elements,
                           rmesh.neighbors, rmesh.boundary_kind)
    og = oracle.precompute_geometry(om, k, reduced_degrees=reduced, g=g, mapping=mapping)
    vol = {q: RM.VolumeGeometry(v.inv_jac, v.jxw) for q, v in og.vol.items()}
    face = {f: RM.FaceGeometry(v.normal, v.jxw) for f, v in og.face.items()}
    return RM.GeometryCache(k, vol, face, og.h_min, og.cartesian_flag)


CASES = [
    # name, d, n, k, boundary, deform amp (x 1/n), material, flux, extra
    ("q2_soft_deformed_k2", 2, 3, 2, "sound_soft", 0.05, "random", {}, {}),
    ("q2_periodic_k3", 2, 4, 3, "periodic", 0.0, "uniform", {}, {}),
    ("q2_soft_sheared_k5", 2, 3, 5, "sound_soft", 0.0, "random", {}, {"shear": True}),
    ("h3_periodic_deformed_k3", 3, 2, 3, "periodic", 0.05, "random", {}, {}),
    ("h3_soft_k4", 3, 3, 4, "sound_soft", 0.0, "random", {}, {}),
    ("h3_periodic_k7", 3, 2, 7, "periodic", 0.0, "uniform", {}, {}),
    ("h3_soft_deformed_k2_tau", 3, 2, 2, "sound_soft", 0.04, "random", {"tau": 0.7}, {}),
    ("h3_periodic_k3_nostab", 3, 2, 3, "periodic", 0.0, "random",
     {"stabilization": False}, {}),
    ("h3_soft_sheared_k3", 3, 2, 3, "sound_soft", 0.0, "random", {}, {"shear": True}),
    ("h3_curved_k5", 3, 2, 5, "periodic", 0.0, "random", {}, {"curved": True}),
]


def operator_case(name, d, n, k, boundary, amp, matkind, flux, extra, seed):
    rng = np.random.default_rng(seed)
    rmesh = RM.build_cartesian(n, d, boundary)
    if amp:
        rmesh = RM.deform(rmesh, amp / n)
    if extra.get("shear"):
        T = np.eye(d) + 0.25 * rng.standard_normal((d, d))
        rmesh = dataclasses.replace(rmesh, vertices=rmesh.vertices @ T.T)
    reduced = tuple(sorted({q for p in ("every_second", "every_step", "every_third")
                            for q in RS.reduction_degrees(k, p)}, reverse=True))
    if extra.get("curved"):
        geo = _oracle_geometry(rmesh, k, 5, configs.c3_mapping, reduced)
    else:
        geo = RM.precompute_geometry(rmesh, k, reduced_degrees=reduced)
    E = rmesh.n_elements
    if matkind == "random":
        mat = RM.Material(c=rng.uniform(0.5, 2.0, E), rho=rng.uniform(0.5, 2.0, E))
    else:
        mat = RM.Material.uniform(rmesh)
    fp = FluxParams(**flux)
    op = RO.AcousticOperator(rmesh, geo, mat, flux=fp)
    u = rng.standard_normal((E, d + 1) + (k + 1,) * d)
    st = StateVector(u, k, d)
    dt = 0.3 * RS.compute_dt(0.2, rmesh, mat, k) if extra.get("curved") else 0.01
    out = dict(d=d, k=k, boundary=boundary, vertices=rmesh.vertices,
               elements=rmesh.elements, neighbors=rmesh.neighbors,
               n_per_dim=np.array(rmesh.n_per_dim), c=mat.c, rho=mat.rho,
               tau=np.nan if fp.tau is None else fp.tau,
               stabilization=int(fp.stabilization), u=u, dt=dt,
               curved=int(bool(extra.get("curved"))), reduced=np.array(reduced, dtype=int))
    out["K_both"] = op.apply_K(st).data
    out["K_cell"] = op.apply_K(st, "cell").data
    out["K_face"] = op.apply_K(st, "face").data
    out["Minv"] = op.apply_inverse_mass(st).data
    out["M"] = op.apply_mass(st).data
    out["rhs"] = op.rhs(st).data
    vals = op.to_gauss_values(u)
    out["to_gauss"] = vals
    out["from_gauss_weighted"] = op.from_gauss_weighted(vals)
    out["localS_k"] = op.apply_local_S(vals, k)
    for q in reduced:
        vq = rng.standard_normal((E, d + 1) + (q + 1,) * d)
        out[f"localS_in_{q}"] = vq
        out[f"localS_{q}"] = op.apply_local_S(vq, q)
        if q < k:
            out[f"resize_down_{q}"] = op.resize_values(vals, k, q)
            out[f"resize_up_{q}"] = op.resize_values(vq, q, k)
    for pol in ("none", "every_second", "every_step", "every_third"):
        for sh in (False, True):
            out[f"tck_{pol}_{int(sh)}"] = RS.tck_evaluate(st, dt, op, pol, sh).data
    for var in ("ader", "ader_hdg"):
        for pol in ("none", "every_second"):
            out[f"ader_{var}_{pol}"] = RS.ader_step(st, dt, op, var, pol).data
    out["lsrk45"] = RS.lsrk_step(st, dt, RS.LSRK45, op).data
    out["lsrk59"] = RS.lsrk_step(st, dt, RS.LSRK59, op).data
    out["rk4"] = RS.rk_step(st, dt, RS.RK4_CLASSIC, op).data
    out["norm"] = RS.state_norm(op, st)
    np.savez_compressed(os.path.join(HERE, f"op_{name}.npz"), **out)


TRAJ = [
    # name, config, scale, scheme, steps
    ("c1_lsrk45_10", "c1", 1.0, "lsrk45", 10),
    ("c2s_lsrk45_100", "c2", 0.125, "lsrk45", 100),
    ("c3s_ader_hdg_10", "c3", 0.0625, "ader_hdg", 10),
    ("c4s_ader_hdg_20", "c4", 1 / 24, "ader_hdg", 20),
    ("c4s_lsrk45_20", "c4", 1 / 24, "lsrk45", 20),
    ("c5s_lsrk45_20", "c5", 1 / 32, "lsrk45", 20),
    ("c5s_ader_hdg_20", "c5", 1 / 32, "ader_hdg", 20),
]


def trajectory(name, cfg, scale, scheme, steps):
    prob = configs.config(cfg, scale=scale)
    m = prob.mesh
    rmesh = RM.Mesh(m.d, m.n_per_dim, m.vertices, m.elements, m.neighbors, [],
                    m.boundary_kind)
    k = prob.k
    reduced = RS.reduction_degrees(k, "every_second")
    if cfg == "c3":
        base = RM.build_cartesian(m.n_per_dim, 3, "periodic")
        geo = _oracle_geometry(base, k, 5, configs.c3_mapping, reduced)
    else:
        geo = RM.precompute_geometry(rmesh, k, reduced_degrees=reduced)
    mat = RM.Material(c=prob.material.c, rho=prob.material.rho)
    op = RO.AcousticOperator(rmesh, geo, mat)
    cr = prob.schemes[scheme][0]
    dt = RS.compute_dt(cr, rmesh, mat, k)
    stepper = RS.make_stepper(RS.SchemeConfig(scheme=scheme, courant=cr), op)
    st = RS.advance(StateVector(prob.state.copy(), k, m.d), dt, steps, stepper)
    np.savez_compressed(os.path.join(HERE, f"traj_{name}.npz"), config=cfg, scale=scale,
                        scheme=scheme, steps=steps, dt=dt, courant=cr, u0=prob.state,
                        u_final=st.data)


if __name__ == "__main__":
    # optional arguments: names of the cases to (re)generate (default: all)
    only = set(sys.argv[1:])
    if not only or "tables" in only:
        tables()
    for i, case in enumerate(CASES):
        if not only or case[0] in only:
            print("op", case[0], flush=True)
            operator_case(*case, seed=1000 + i)
    for t in TRAJ:
        if not only or t[0] in only:
            print("traj", t[0], flush=True)
            trajectory(*t)
    print("reference version", getattr(wavekernel, "__version__", "0.1.0"))
