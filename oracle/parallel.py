"""Multi-threaded driver of the oracle operator (test infrastructure / CPU
baseline only).

``bench.py --impl reference`` times the reference algorithm on the GPU box's
host cores "with all the host threads it can use".  The restated operator is
element-local except for the face traces, so the element range is split into
chunks evaluated by a thread pool (numpy releases the GIL inside its BLAS
contractions and large ufuncs).  Results are identical to the single-threaded
oracle up to floating-point association within BLAS.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .mesh import OracleGeometry, OracleMaterial, OracleMesh, FaceMetric, VolumeMetric
from .operator import OracleOperator


def _sub_operator(op: OracleOperator, lo: int, hi: int) -> OracleOperator:
    """Operator restricted to elements [lo, hi): neighbours keep global ids."""
    g = op.geometry
    vol = {q: VolumeMetric(v.inv_jac[lo:hi], v.jxw[lo:hi]) for q, v in g.vol.items()}
    face = {f: FaceMetric(v.normal[lo:hi], v.jxw[lo:hi]) for f, v in g.face.items()}
    geo = OracleGeometry(g.degree, vol, face, g.h_min, g.cartesian_flag[lo:hi])
    m = op.mesh
    mesh = OracleMesh(m.d, m.n_per_dim, m.vertices, m.elements[lo:hi], m.neighbors[lo:hi],
                      m.boundary_kind)
    mat = OracleMaterial(np.asarray(op.material.c)[lo:hi], np.asarray(op.material.rho)[lo:hi])
    sub = OracleOperator(mesh, geo, mat, stabilization=op.stabilization)
    sub.tau = op.tau[lo:hi]
    return sub


class ThreadedOracle:
    """rhs / LSRK stage of the oracle evaluated chunk-parallel."""

    def __init__(self, op: OracleOperator, n_threads: int | None = None):
        self.op = op
        self.n_threads = n_threads or os.cpu_count() or 1
        E = op.mesh.n_elements
        bounds = np.linspace(0, E, self.n_threads + 1).astype(int)
        self.chunks = [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        self.subs = [_sub_operator(op, a, b) for a, b in self.chunks]
        self.pool = ThreadPoolExecutor(max_workers=len(self.chunks))

    def _rhs_chunk(self, i, u, out):
        lo, hi = self.chunks[i]
        sub = self.subs[i]
        d = self.op.d
        r = sub._cell(u[lo:hi])
        # faces: own traces from the chunk, neighbour traces from the full state
        r += self._faces(sub, u, lo, hi)
        out[lo:hi] = -sub.apply_inverse_mass(r)

    def _faces(self, sub, u, lo, hi):
        # evaluate the face term of elements [lo, hi) with global neighbour ids
        op = self.op
        full = u
        local = u[lo:hi]
        # temporarily view neighbours through a remapped state: gather the
        # neighbour elements needed into a compact array
        nbr = sub.mesh.neighbors
        need = np.unique(nbr[nbr >= 0])
        remap = -np.ones(op.mesh.n_elements, dtype=np.int64)
        ext = np.concatenate([np.arange(lo, hi), need[(need < lo) | (need >= hi)]])
        remap[ext] = np.arange(ext.size)
        gathered = full[ext]
        nb2 = np.where(nbr >= 0, remap[np.maximum(nbr, 0)], -1)
        mesh2 = OracleMesh(sub.mesh.d, sub.mesh.n_per_dim, sub.mesh.vertices,
                           sub.mesh.elements, nb2, sub.mesh.boundary_kind)
        saved = sub.mesh
        sub.mesh = mesh2
        try:
            r = sub._faces_ext(local, gathered)
        finally:
            sub.mesh = saved
        return r

    def rhs(self, u: np.ndarray) -> np.ndarray:
        out = np.empty_like(u)
        list(self.pool.map(lambda i: self._rhs_chunk(i, u, out), range(len(self.chunks))))
        return out

    def lsrk_step(self, u: np.ndarray, dt: float, scheme: dict) -> np.ndarray:
        u = u.copy()
        r = np.zeros_like(u)
        for a, b in zip(scheme["a"], scheme["b"]):
            f = self.rhs(u)
            r = r * a + f * dt
            u = u + r * b
        return u

    def close(self):
        self.pool.shutdown()
