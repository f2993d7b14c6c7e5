"""Shared test helpers: load golden cases into oracle / product objects."""

from __future__ import annotations

import glob
import os

import numpy as np

import oracle
from oracle import stepping as OS

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    den = np.linalg.norm(ref)
    return np.linalg.norm(got - ref) / (den if den > 0 else 1.0)


def op_cases():
    return sorted(os.path.basename(p)[3:-4] for p in glob.glob(os.path.join(GOLDEN, "op_*.npz")))


def traj_cases():
    return sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(GOLDEN, "traj_*.npz")))


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))


class Case:
    """A golden operator case rebuilt as oracle objects (and, lazily, GPU ones)."""

    def __init__(self, name):
        self.name = name
        z = load("op_" + name)
        self.z = z
        self.d, self.k = int(z["d"]), int(z["k"])
        self.mesh = oracle.OracleMesh(self.d, tuple(int(v) for v in z["n_per_dim"]),
                                      z["vertices"], z["elements"], z["neighbors"],
                                      str(z["boundary"]))
        self.curved = bool(int(z["curved"]))
        reduced = tuple(int(v) for v in z["reduced"])
        if self.curved:
            from paper_1805_03981_b200.configs import c3_mapping
            base = oracle.build_cartesian(self.mesh.n_per_dim, self.d, self.mesh.boundary_kind)
            self.geometry = oracle.precompute_geometry(base, self.k, reduced, g=5,
                                                       mapping=c3_mapping)
        else:
            self.geometry = oracle.precompute_geometry(self.mesh, self.k, reduced)
        self.material = oracle.OracleMaterial(z["c"], z["rho"])
        tau = float(z["tau"])
        self.tau = None if np.isnan(tau) else tau
        self.stab = bool(int(z["stabilization"]))
        self.op = oracle.OracleOperator(self.mesh, self.geometry, self.material,
                                        tau=self.tau, stabilization=self.stab)
        self.u = z["u"]
        self.dt = float(z["dt"])
        self.reduced = reduced

    def gpu_operator(self):
        import paper_1805_03981_b200 as W
        from paper_1805_03981_b200.operator import FluxParams
        return W.AcousticOperator(self.mesh, self.geometry, self.material,
                                  flux=FluxParams(tau=self.tau, stabilization=self.stab))


# ---------------------------------------------------------------------------
# element patches: full-size parity by locality
#
# An output element of the operator depends only on itself and its face
# neighbours (reference operator.py:193-246; the reference test
# tests/test_operator.py:139-147 pins this locality), one ADER-HDG step on the
# elements within face distance 2 (W = M^-1 K U is needed on the
# neighbours).  So a full-size GPU result can be checked element by element
# against the oracle run on a small patch around each sampled element.

def patch(mesh, centers, radius):
    """Elements within face distance ``radius`` of ``centers``; returns
    (global ids, (P, d, 2) patch-local neighbour table, local index of each
    center).  Rim elements whose neighbours lie outside point to themselves
    (their outputs are not compared)."""
    nbr = np.asarray(mesh.neighbors)
    sel = set(int(c) for c in centers)
    front = np.asarray(sorted(sel), dtype=np.int64)
    for _ in range(radius):
        nxt = nbr[front].ravel()
        nxt = np.unique(nxt[nxt >= 0])
        new = [int(v) for v in nxt if int(v) not in sel]
        sel.update(new)
        front = np.asarray(new, dtype=np.int64)
        if front.size == 0:
            break
    ids = np.asarray(sorted(sel), dtype=np.int64)
    g2l = {int(g): i for i, g in enumerate(ids)}
    loc = np.empty(nbr[ids].shape, dtype=np.int64)
    for i, g in enumerate(ids):
        for m in range(nbr.shape[1]):
            for s in range(2):
                v = int(nbr[g, m, s])
                loc[i, m, s] = -1 if v == -1 else g2l.get(v, i)
    return ids, loc, np.asarray([g2l[int(c)] for c in centers], dtype=np.int64)


def restrict_geometry(geo, ids):
    """The rows ``ids`` of a (host or device) GeometryCache as an oracle
    geometry: the oracle then evaluates the operator on exactly the metric
    the GPU used."""
    h = lambda x: x.index_select(0, __import__("torch").as_tensor(ids, device=x.device)).cpu().numpy() \
        if hasattr(x, "index_select") else np.asarray(x)[ids]
    return oracle.OracleGeometry(
        geo.degree, {q: oracle.mesh.VolumeMetric(h(v.inv_jac), h(v.jxw)) for q, v in geo.vol.items()},
        {f: oracle.mesh.FaceMetric(h(v.normal), h(v.jxw)) for f, v in geo.face.items()},
        geo.h_min, np.asarray(geo.cartesian_flag)[ids])


def patch_operator(mesh, ids, loc, k, c, rho, reduced=(), mapping=None, g=1, geometry=None):
    """Oracle operator on a patch (vertices shared with the full mesh);
    ``geometry``: use these metric rows instead of building them."""
    pm = oracle.OracleMesh(mesh.d, tuple(mesh.n_per_dim), np.asarray(mesh.vertices),
                           np.asarray(mesh.elements)[ids], loc, mesh.boundary_kind)
    geo = geometry if geometry is not None else \
        oracle.precompute_geometry(pm, k, reduced, g=g, mapping=mapping)
    mat = oracle.OracleMaterial(np.asarray(c)[ids], np.asarray(rho)[ids])
    return oracle.OracleOperator(pm, geo, mat)
