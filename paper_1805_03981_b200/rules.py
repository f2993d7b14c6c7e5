"""Host-side 1-D rules for input and geometry setup, in numpy extended precision.

The kernels take their 1-D tables from the native library
(``_lib.basis_table``, long double C++).  The host-side SETUP code -- initial
states sampled at the Gauss-Lobatto nodes, geometry nodes of curved maps and
the Lagrange tables of the metric -- uses this module instead, so that
building a problem (``configs``) never needs ``libwk_b200.so`` (the CPU
reference arm of ``bench.py`` must not load the product library).

Points are the reference's rules on [0, 1] (``/root/reference/pkg/src/
wavekernel/quadrature.py:110-154``): Gauss = roots of P_n, Gauss-Lobatto =
{0, 1} and the roots of P'_{n-1}.  They are found by Newton iteration in
``np.longdouble`` (64-bit mantissa) and rounded once; the results are
bit-identical to the native tables for k = 1..12 (tests/test_rules.py).

``lagrange_ld`` evaluates Lagrange value / derivative rows in long double
(the product formula of quadrature.py:157-184); the curved-metric builders
use it so the derivative rows sum to zero far below double round-off (the
metric is then computed from coordinates of size ~1 but Jacobians of size
h).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

LD = np.longdouble


def _legendre(n: int, x):
    """P_n(x) and P_n'(x) by the three-term recurrence (x != +-1)."""
    p0 = np.ones_like(x)
    if n == 0:
        return p0, np.zeros_like(x)
    p1 = x.copy()
    for j in range(2, n + 1):
        p0, p1 = p1, ((2 * j - 1) * x * p1 - (j - 1) * p0) / j
    return p1, n * (x * p1 - p0) / (x * x - 1)


def _newton(f, x):
    for _ in range(100):
        dx = f(x)
        x = x - dx
        if np.max(np.abs(dx)) < LD(1e-30):
            break
    return x


@lru_cache(maxsize=None)
def _gauss_ld(n: int):
    if n < 1:
        raise ValueError("need at least one quadrature point")
    i = np.arange(1, n + 1, dtype=np.float64)
    x = (-np.cos(np.pi * (i - 0.25) / (n + 0.5))).astype(LD)

    def step(x):
        p, dp = _legendre(n, x)
        return p / dp
    x = _newton(step, x)
    x = LD(0.5) * (x - x[::-1])                       # exact mirror symmetry
    _, dp = _legendre(n, x)
    w = LD(2) / ((1 - x * x) * dp * dp)
    return (x + 1) / 2, w / 2


@lru_cache(maxsize=None)
def _gauss_lobatto_ld(n: int):
    if n < 2:
        raise ValueError("Gauss-Lobatto needs n >= 2")
    k = n - 1
    if k == 1:
        return np.array([LD(0), LD(1)]), np.array([LD(0.5), LD(0.5)])
    x = (-np.cos(np.pi * np.arange(1, k, dtype=np.float64) / k)).astype(LD)

    def step(x):
        # roots of P_k': (1 - x^2) P_k'' = 2 x P_k' - k (k + 1) P_k
        p, dp = _legendre(k, x)
        return dp * (1 - x * x) / (2 * x * dp - k * (k + 1) * p)
    x = _newton(step, x)
    x = LD(0.5) * (x - x[::-1])
    xx = np.concatenate(([LD(-1)], x, [LD(1)]))
    p = np.array([_legendre(k, np.array([v]))[0][0] if abs(v) != 1 else LD(1) for v in xx])
    w = LD(2) / (k * (k + 1) * p * p)
    pts = (xx + 1) / 2
    pts[0], pts[-1] = LD(0), LD(1)
    return pts, w / 2


def gauss_points(k: int) -> np.ndarray:
    return _gauss_ld(k + 1)[0].astype(np.float64)


def gauss_weights(k: int) -> np.ndarray:
    return _gauss_ld(k + 1)[1].astype(np.float64)


def gl_points(k: int) -> np.ndarray:
    return _gauss_lobatto_ld(k + 1)[0].astype(np.float64)


def lagrange_ld(nodes, pts, derivative: bool = False) -> np.ndarray:
    """mat[i, j] = L_j(pts_i) (or L_j'(pts_i)) in long double, for DOUBLE
    ``nodes`` / ``pts`` (the rows of the interpolant of the rounded nodes)."""
    nodes = np.asarray(nodes, dtype=np.float64).astype(LD)
    pts = np.asarray(pts, dtype=np.float64).astype(LD)
    n = nodes.size
    out = np.zeros((pts.size, n), dtype=LD)
    for j in range(n):
        others = np.delete(nodes, j)
        den = np.prod(nodes[j] - others)
        if not derivative:
            out[:, j] = np.prod(pts[:, None] - others[None, :], axis=1) / den
        else:
            for r in range(n - 1):
                rest = np.delete(others, r)
                out[:, j] += np.prod(pts[:, None] - rest[None, :], axis=1)
            out[:, j] /= den
    return out
