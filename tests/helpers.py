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
