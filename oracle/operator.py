"""Oracle restatement of the reference matrix-free operator (test infrastructure).

Follows ``/root/reference/pkg/src/wavekernel/operator.py``.  States are
plain arrays of shape (E, d+1, n, ..., n) in the GL basis with components
v_1..v_d, p and direction 0 on the last axis (operator.py:33-55).

The arithmetic is the reference's: the split strong/weak cell form
(operator.py:149-191), element-wise HDG/upwind face terms with the OWN
element's coefficients and the sound-soft mirror (operator.py:206-246),
the basis-change mass inverse (operator.py:250-258), and the collocated
local operators of the Taylor loop (operator.py:276-325).  It is written
as whole-mesh tensor contractions (``_along``) instead of the
reference's ``apply_1d`` loop.
"""

from __future__ import annotations

import numpy as np

from . import quadrature as Q


def _along(mat: np.ndarray, arr: np.ndarray, m: int) -> np.ndarray:
    """Mode-m product: direction m is axis ndim-1-m (kernels.py:108-143)."""
    ax = arr.ndim - 1 - m
    return np.moveaxis(np.tensordot(arr, mat, axes=([ax], [1])), -1, ax)


def _along_all(mat: np.ndarray, arr: np.ndarray, ndir: int) -> np.ndarray:
    for m in range(ndir):
        arr = _along(mat, arr, m)
    return arr


class OracleOperator:
    """K, M^{-1}, M, rhs and the local Taylor-loop operators on one mesh."""

    def __init__(self, mesh, geometry, material, tau=None, stabilization=True):
        if geometry.cartesian_flag.shape[0] != mesh.n_elements:
            raise ValueError("geometry was built for a different mesh")
        self.mesh, self.geometry, self.material = mesh, geometry, material
        self.d = mesh.d
        self.k = geometry.degree
        self.n_comp = self.d + 1
        self.stabilization = stabilization
        k, e = self.k, mesh.n_elements
        self.B, self.Binv = Q.basis_change(k)
        self.dgl = Q.gl_derivative_at_gauss(k)
        self.inv_rho = 1.0 / np.asarray(material.rho, dtype=float)
        self.c2rho = np.asarray(material.c, dtype=float) ** 2 * np.asarray(material.rho, dtype=float)
        if tau is None:
            self.tau = 1.0 / (np.asarray(material.c) * np.asarray(material.rho))
        else:
            self.tau = np.full(e, float(tau))
        if np.any(self.tau <= 0):
            raise ValueError("stabilization must be positive")

    # broadcasting helpers
    def _e(self, v, extra):
        return v.reshape((-1,) + (1,) * extra)

    def check(self, u: np.ndarray):
        expect = (self.mesh.n_elements, self.n_comp) + (self.k + 1,) * self.d
        if u.shape != expect:
            raise ValueError(f"state shape {u.shape}, expected {expect}")

    # -- K: operator.py:149-191 ------------------------------------------
    def apply_K(self, u: np.ndarray, parts: str = "both") -> np.ndarray:
        self.check(u)
        d, k = self.d, self.k
        r = np.zeros_like(u)
        if parts in ("both", "cell"):
            r += self._cell(u)
        if parts in ("both", "face"):
            r += self._faces(u)
        return r

    def _cell(self, u):
        d, k = self.d, self.k
        vm = self.geometry.vol[k]
        G, jxw = vm.inv_jac, vm.jxw                      # (E,d,d,q..), (E,q..)
        uq = _along_all(self.B, u, d)                    # Gauss values
        # reference-coordinate gradients at the Gauss points via d_gl
        grads = []
        for m in range(d):
            g = u
            for j in range(d):
                g = _along(self.dgl if j == m else self.B, g, j)
            grads.append(g)
        half_v = 0.5 * jxw * self._e(self.inv_rho, d)
        half_p = 0.5 * jxw * self._e(self.c2rho, d)
        strong = np.zeros_like(u)
        for i in range(d):
            strong[:, i] = half_v * sum(G[:, m, i] * grads[m][:, d] for m in range(d))
        strong[:, d] = half_p * sum(G[:, m, i] * grads[m][:, i]
                                    for m in range(d) for i in range(d))
        weak = np.zeros_like(u)
        dco_t = Q.collocation_derivative(k).T
        for m in range(d):
            flux = np.empty_like(u)
            for i in range(d):
                flux[:, i] = -half_v * G[:, m, i] * uq[:, d]
            flux[:, d] = -half_p * sum(G[:, m, i] * uq[:, i] for i in range(d))
            weak += _along(dco_t, flux, m)
        return _along_all(self.B.T, strong + weak, d)

    # -- faces: operator.py:193-246 --------------------------------------
    def _slice(self, m, side):
        idx = [slice(None)] * (2 + self.d)
        idx[2 + self.d - 1 - m] = -1 if side else 0
        return tuple(idx)

    def _faces(self, u):
        return self._faces_ext(u, u)

    def _faces_ext(self, u, u_nbr):
        """Face term of the elements of ``u``; neighbour ids index ``u_nbr``."""
        d = self.d
        r = np.zeros_like(u)
        # face-node GL coefficients -> face Gauss values, d-1 sweeps
        tr = {(m, s): _along_all(self.B, u[self._slice(m, s)], d - 1)
              for m in range(d) for s in (0, 1)}
        trn = tr if u_nbr is u else {
            (m, s): _along_all(self.B, u_nbr[self._slice(m, s)], d - 1)
            for m in range(d) for s in (0, 1)}
        ext = d - 1
        ir, c2r, tau = (self._e(self.inv_rho, ext), self._e(self.c2rho, ext),
                        self._e(self.tau, ext))
        for m in range(d):
            for s in (0, 1):
                own = tr[(m, s)]
                nbr = self.mesh.neighbors[:, m, s]
                other = trn[(m, 1 - s)][np.where(nbr >= 0, nbr, 0)].copy()
                wall = nbr < 0
                other[wall, :d] = own[wall, :d]        # sound-soft mirror
                other[wall, d] = -own[wall, d]
                fm = self.geometry.face[(m, s)]
                nrm = fm.normal
                vn_o = sum(nrm[:, i] * own[:, i] for i in range(d))
                vn_x = sum(nrm[:, i] * other[:, i] for i in range(d))
                pv = 0.5 * ir * other[:, d]
                pp = 0.5 * c2r * vn_x
                if self.stabilization:
                    pv = pv + 0.5 * ir / tau * (vn_o - vn_x)
                    pp = pp + 0.5 * c2r * tau * (own[:, d] - other[:, d])
                integ = np.concatenate([(pv * nrm[:, i])[:, None] for i in range(d)]
                                       + [pp[:, None]], axis=1)
                integ = integ * fm.jxw[:, None]
                r[self._slice(m, s)] += _along_all(self.B.T, integ, d - 1)
        return r

    # -- mass: operator.py:250-272 -----------------------------------------
    def apply_inverse_mass(self, x: np.ndarray) -> np.ndarray:
        self.check(x)
        jxw = self.geometry.vol[self.k].jxw
        t = _along_all(self.Binv.T, x, self.d) / jxw[:, None]
        return _along_all(self.Binv, t, self.d)

    def apply_mass(self, x: np.ndarray) -> np.ndarray:
        self.check(x)
        jxw = self.geometry.vol[self.k].jxw
        t = _along_all(self.B, x, self.d) * jxw[:, None]
        return _along_all(self.B.T, t, self.d)

    def rhs(self, u: np.ndarray) -> np.ndarray:
        return -self.apply_inverse_mass(self.apply_K(u))

    # -- collocated Taylor-loop pieces: operator.py:276-325 ----------------
    def to_gauss_values(self, u: np.ndarray) -> np.ndarray:
        return _along_all(self.B, u, self.d)

    def from_gauss_weighted(self, vals: np.ndarray) -> np.ndarray:
        jxw = self.geometry.vol[self.k].jxw
        return _along_all(self.B.T, vals * jxw[:, None], self.d)

    def apply_local_S(self, vals: np.ndarray, degree: int) -> np.ndarray:
        if degree not in self.geometry.vol:
            raise ValueError(f"geometry has no degree-{degree} point set")
        d = self.d
        G = self.geometry.vol[degree].inv_jac
        dco = Q.collocation_derivative(degree)
        grads = [_along(dco, vals, m) for m in range(d)]
        out = np.empty_like(vals)
        for i in range(d):
            out[:, i] = self._e(self.inv_rho, d) * sum(G[:, m, i] * grads[m][:, d]
                                                       for m in range(d))
        out[:, d] = self._e(self.c2rho, d) * sum(G[:, m, i] * grads[m][:, i]
                                                 for m in range(d) for i in range(d))
        return out

    def resize_values(self, vals: np.ndarray, k_from: int, k_to: int) -> np.ndarray:
        if k_from == k_to:
            return vals
        return _along_all(Q.resize_matrix(k_from, k_to), vals, self.d)
