"""Oracle restatement of the reference time integrators (test infrastructure).

Follows ``/root/reference/pkg/src/wavekernel/stepping.py`` (LSRK
coefficients :88-143, ``lsrk_step`` :179-207, ``tck_evaluate`` :215-262,
``ader_step`` :265-285, ``compute_dt`` :311-318, ``state_norm`` :321-324)
and ``kernels.py:286-309`` (degree-reduction schedule).  The scheme
coefficients are data of the published schemes and are reproduced
exactly, since parity depends on them.
"""

from __future__ import annotations

import math

import numpy as np

from .mesh import min_edge_length

# Carpenter-Kennedy (1994) five-stage fourth-order 2N scheme (stepping.py:88-106)
LSRK45 = dict(
    name="lsrk45",
    a=(0.0, -567301805773 / 1357537059087, -2404267990393 / 2016746695238,
       -3550918686646 / 2091501179385, -1275806237668 / 842570457699),
    b=(1432997174477 / 9575080441755, 5161836677717 / 13612068292357,
       1720146321549 / 2090206949498, 3134564353537 / 4481467310338,
       2277821191437 / 14882151754819),
)

# The reference's nine-stage register weights (stepping.py:113-143)
LSRK59 = dict(
    name="lsrk59",
    a=(0.0, -0.6304365496865543, -1.1303843359562102, -0.3293878463661334,
       -1.4487682419993357, -0.8130202966406633, -0.9436317245996502,
       -0.058029253696775494, -1.2209100426892907),
    b=(0.03321496462492457, 0.5563858748215249, 0.721229659783645,
       0.0770373034268954, 0.7269522462792919, 0.27832474096203197,
       0.19393254670497226, 0.16876385757079637, 0.304085932161835),
)

_STRIDE = {"none": 0, "every_step": 1, "every_second": 2, "every_third": 3}


def reduction_schedule(k: int, policy: str):
    """(deg_in, deg_out) per Taylor application j = 1..k+1 (kernels.py:286-302)."""
    s = _STRIDE[policy]
    out, deg = [], k
    for j in range(1, k + 2):
        nxt = max(deg - s, 0) if (s and j % s == 0) else deg
        out.append((deg, nxt))
        deg = nxt
    return out


def reduction_degrees(k: int, policy: str):
    """Reduced degrees a policy visits, descending (kernels.py:305-309)."""
    return tuple(sorted({o for _, o in reduction_schedule(k, policy)} - {k}, reverse=True))


def lsrk_step(u: np.ndarray, dt: float, scheme: dict, op) -> np.ndarray:
    """Two-register 2N step (stepping.py:179-207), merged-update arithmetic."""
    u = u.copy()
    r = np.zeros_like(u)
    for a, b in zip(scheme["a"], scheme["b"]):
        f = op.rhs(u)
        r = r * a + f * dt
        u = u + r * b
    return u


def taylor_weight(j: int, dt: float) -> float:
    """(-1)^j dt^{j+1} / (j+1)! (stepping.py:210-212)."""
    return (-1.0 if j % 2 else 1.0) * dt ** (j + 1) / math.factorial(j + 1)


def tck_evaluate(u: np.ndarray, dt: float, op, reduction: str = "every_second",
                 shift: bool = False) -> np.ndarray:
    """Element-local Taylor sum, mass-weighted GL output (stepping.py:215-262)."""
    op.check(u)
    k = op.k
    cur = op.to_gauss_values(u)
    acc = {k: taylor_weight(1 if shift else 0, dt) * cur}
    sched = reduction_schedule(k, reduction)
    n_apps = max(k - 1, 0) if shift else k + 1
    deg = k
    for j in range(1, n_apps + 1):
        d_in, d_out = sched[j - 1]
        if d_in == 0:
            break
        cur = op.apply_local_S(cur, deg)
        if d_out != d_in:
            cur = op.resize_values(cur, d_in, d_out)
            deg = d_out
        w = taylor_weight(j + 1 if shift else j, dt)
        acc[deg] = acc[deg] + w * cur if deg in acc else w * cur
    degs = sorted(acc)
    for lo in degs:
        if lo == k:
            break
        hi = min(q for q in acc if q > lo)
        acc[hi] = acc[hi] + op.resize_values(acc[lo], lo, hi)
    return op.from_gauss_weighted(acc[k])


def ader_step(u: np.ndarray, dt: float, op, variant: str = "ader_hdg",
              reduction: str = "every_second") -> np.ndarray:
    """One ADER step (stepping.py:265-285)."""
    if variant == "ader":
        y = op.apply_inverse_mass(tck_evaluate(u, dt, op, reduction))
        return u - op.apply_inverse_mass(op.apply_K(y))
    if variant == "ader_hdg":
        w = op.apply_inverse_mass(op.apply_K(u))
        y = op.apply_inverse_mass(tck_evaluate(w, dt, op, reduction, shift=True))
        z = op.apply_inverse_mass(op.apply_K(y))
        return u - dt * w - z
    raise ValueError(f"unknown ader variant {variant!r}")


def advance(u, dt, n_steps, step):
    for _ in range(n_steps):
        u = step(u, dt)
    return u


def compute_dt(courant: float, mesh, material, k: int) -> float:
    """dt = Cr h_min / (c_max k^1.5) (stepping.py:311-318)."""
    if courant <= 0.0:
        raise ValueError("Courant number must be positive")
    return courant * min_edge_length(mesh) / (float(np.max(material.c)) * max(k, 1) ** 1.5)


def state_norm(op, u: np.ndarray) -> float:
    """Mass-weighted discrete L2 norm (stepping.py:321-324)."""
    return float(np.sqrt(abs(np.vdot(u, op.apply_mass(u)))))
