"""Oracle restatement of the reference 1-D bases (test infrastructure).

Follows ``/root/reference/pkg/src/wavekernel/quadrature.py``; all rules
live on [0, 1].  The algorithms are restated, not copied: Gauss-Lobatto
points come from the roots of P'_{n-1} (numpy's Legendre class) instead
of the reference's Newton loop, and Lagrange matrices use the
barycentric form instead of the product formula.  Both agree with the
reference to round-off; ``tests/test_oracle_golden.py`` pins them
against the reference's tables.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np
from numpy.polynomial import legendre as npleg


@lru_cache(maxsize=None)
def gauss_rule(n: int) -> tuple[np.ndarray, np.ndarray]:
    """n-point Gauss-Legendre rule on [0,1] (reference quadrature.py:110-115)."""
    if n < 1:
        raise ValueError("need at least one quadrature point")
    x, w = npleg.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


@lru_cache(maxsize=None)
def gauss_lobatto_rule(n: int) -> tuple[np.ndarray, np.ndarray]:
    """n-point Gauss-Lobatto rule on [0,1] (reference quadrature.py:118-154).

    Interior points are the roots of P'_{n-1}; weights are
    2 / (n (n-1) P_{n-1}(x)^2) on [-1,1], halved for [0,1].
    """
    if n < 2:
        raise ValueError("Gauss-Lobatto needs n >= 2")
    pn1 = npleg.Legendre.basis(n - 1)
    interior = np.sort(np.real(pn1.deriv().roots())) if n > 2 else np.zeros(0)
    # one Newton polish of the interior roots on P'_{n-1}
    if n > 2:
        d1, d2 = pn1.deriv(1), pn1.deriv(2)
        interior = interior - d1(interior) / d2(interior)
        interior = 0.5 * (interior - interior[::-1])  # exact mirror symmetry
    x = np.concatenate(([-1.0], interior, [1.0]))
    w = 2.0 / (n * (n - 1) * pn1(x) ** 2)
    pts = 0.5 * (x + 1.0)
    pts[0], pts[-1] = 0.0, 1.0
    return pts, 0.5 * w


def _bary_weights(nodes: np.ndarray) -> np.ndarray:  # noqa: D401
    diff = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff, 1.0)
    return 1.0 / np.prod(diff, axis=1)


def lagrange_matrix(nodes, points, kind: str = "value", dtype=float) -> np.ndarray:
    """mat[i, j] = L_j(points_i) or L_j'(points_i) for the Lagrange basis on
    ``nodes`` (reference quadrature.py:157-184), barycentric evaluation.

    ``dtype=np.longdouble`` evaluates the rows of the (double) nodes in
    extended precision (used by the curved-metric restatement, mesh.py)."""
    nodes = np.asarray(nodes, dtype=float).astype(dtype)
    pts = np.asarray(points, dtype=float).astype(dtype)
    if kind not in ("value", "derivative"):
        raise ValueError(f"unknown kind {kind!r}")
    nn = nodes.size
    lam = _bary_weights(nodes)
    out = np.empty((pts.size, nn), dtype=dtype)
    for i, x in enumerate(pts):
        hit = np.nonzero(np.abs(x - nodes) < 1e-14)[0]
        if kind == "value":
            if hit.size:
                out[i] = 0.0
                out[i, hit[0]] = 1.0
            else:
                t = lam / (x - nodes)
                out[i] = t / t.sum()
            continue
        if hit.size:
            # derivative at a node: D_ij = (lam_j/lam_q)/(x_q-x_j), D_qq = -sum
            q = hit[0]
            row = np.zeros(nn, dtype=dtype)
            others = np.arange(nn) != q
            row[others] = (lam[others] / lam[q]) / (nodes[q] - nodes[others])
            row[q] = -row[others].sum()
            out[i] = row
        else:
            # d/dx of l(x) * lam_j/(x-x_j), l(x) = prod (x - x_m)
            dx = x - nodes
            ell = np.prod(dx)
            s1 = np.sum(1.0 / dx)
            out[i] = ell * lam / dx * (s1 - 1.0 / dx)
    return out


@lru_cache(maxsize=None)
def basis_change(k: int) -> tuple[np.ndarray, np.ndarray]:
    """(GL->Gauss, Gauss->GL) value matrices (reference quadrature.py:239-254)."""
    if k == 0:
        one = np.ones((1, 1))
        return one, one
    gl, _ = gauss_lobatto_rule(k + 1)
    g, _ = gauss_rule(k + 1)
    return lagrange_matrix(gl, g), lagrange_matrix(g, gl)


@lru_cache(maxsize=None)
def gl_derivative_at_gauss(k: int) -> np.ndarray:
    """d_gl: derivative of the GL basis at the Gauss points (operator.py:111)."""
    gl, _ = gauss_lobatto_rule(k + 1)
    g, _ = gauss_rule(k + 1)
    return lagrange_matrix(gl, g, "derivative")


@lru_cache(maxsize=None)
def collocation_derivative(k: int) -> np.ndarray:
    """Gauss-nodal derivative at its own points (kernels.py:153-157)."""
    g, _ = gauss_rule(k + 1)
    return lagrange_matrix(g, g, "derivative")


@lru_cache(maxsize=None)
def projection_matrix(k_from: int, k_to: int) -> np.ndarray:
    """L2 projection between Gauss-collocated degrees (quadrature.py:221-236).

    P = W_to^{-1} A_to^T W_mix A_from with the mixed integrals evaluated by
    the (k_from+1)-point Gauss rule, exact for the degree k_from+k_to
    integrand.
    """
    if not 0 <= k_to <= k_from:
        raise ValueError("need 0 <= k_to <= k_from")
    g_to, w_to = gauss_rule(k_to + 1)
    g_from, _ = gauss_rule(k_from + 1)
    x_mix, w_mix = gauss_rule(k_from + 1)
    a_to = lagrange_matrix(g_to, x_mix)
    a_from = lagrange_matrix(g_from, x_mix)
    return (a_to.T * w_mix[None, :]) @ a_from / w_to[:, None]


@lru_cache(maxsize=None)
def interpolation_up(k_from: int, k_to: int) -> np.ndarray:
    """Gauss(k_from) -> Gauss(k_to) interpolation (operator.py:314-315)."""
    g_from, _ = gauss_rule(k_from + 1)
    g_to, _ = gauss_rule(k_to + 1)
    return lagrange_matrix(g_from, g_to)


def resize_matrix(k_from: int, k_to: int) -> np.ndarray:
    """Projection down or interpolation up (operator.py:308-325)."""
    if k_to < k_from:
        return projection_matrix(k_from, k_to)
    return interpolation_up(k_from, k_to)
