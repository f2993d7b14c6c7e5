"""Oracle restatement of the reference mesh/geometry data (test infrastructure).

Follows ``/root/reference/pkg/src/wavekernel/mesh.py``:

* element order e = i0 + n0 (i1 + n1 i2), vertex bit j = high side along
  direction j (mesh.py:69-127);
* ``neighbors[e, axis, side]`` with side 0 = low face, -1 = sound-soft,
  periodic wrap (mesh.py:96-107);
* volume metric ``inv_jac[e, a, b, ...] = d xi_a / d x_b`` and
  ``jxw = det J * w`` at the Gauss points of each degree (mesh.py:245-262);
* face normal ``sgn det J^{-T} e_axis / |.|`` and face JxW
  ``|det J^{-T} e_axis| w`` (mesh.py:265-286).

Restated differently from the reference: the element map is always a
tensor-product Lagrange interpolant on Gauss-Lobatto geometry nodes of
degree ``g``.  With g = 1 the GL nodes are the two endpoints, so this is
exactly the reference's multilinear vertex map; with g > 1 it is the
isoparametric curved map that BASELINE config 3 needs and the reference
mesh code cannot build.  The unchanged reference
``AcousticOperator`` consumes the resulting geometry (it only reads
``vol``, ``face``, ``degree`` and ``cartesian_flag``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .quadrature import gauss_lobatto_rule, gauss_rule, lagrange_matrix


@dataclass(frozen=True)
class OracleMesh:
    d: int
    n_per_dim: tuple
    vertices: np.ndarray
    elements: np.ndarray
    neighbors: np.ndarray
    boundary_kind: str

    @property
    def n_elements(self) -> int:
        return self.elements.shape[0]


@dataclass(frozen=True)
class OracleMaterial:
    """Element-wise constant c, rho (reference mesh.py:145-159)."""
    c: np.ndarray
    rho: np.ndarray

    @classmethod
    def uniform(cls, n_elements: int, c: float = 1.0, rho: float = 1.0):
        return cls(np.full(n_elements, float(c)), np.full(n_elements, float(rho)))


@dataclass(frozen=True)
class VolumeMetric:
    inv_jac: np.ndarray
    jxw: np.ndarray


@dataclass(frozen=True)
class FaceMetric:
    normal: np.ndarray
    jxw: np.ndarray


@dataclass(frozen=True)
class OracleGeometry:
    """Same attribute layout as the reference GeometryCache (mesh.py:162-188)."""
    degree: int
    vol: dict
    face: dict
    h_min: float
    cartesian_flag: np.ndarray = field(repr=False)


def build_cartesian(n_per_dim, d: int, boundary_kind: str = "sound_soft") -> OracleMesh:
    """Uniform structured mesh of [0,1]^d (reference mesh.py:69-127)."""
    if d not in (2, 3):
        raise ValueError("dimension must be 2 or 3")
    if boundary_kind not in ("sound_soft", "periodic"):
        raise ValueError(f"unknown boundary kind {boundary_kind!r}")
    nn = (int(n_per_dim),) * d if np.isscalar(n_per_dim) else tuple(int(v) for v in n_per_dim)
    if len(nn) != d or min(nn) < 1:
        raise ValueError("bad element counts")
    # vertex grid, direction 0 fastest
    axes = [np.linspace(0.0, 1.0, n + 1) for n in nn]
    grids = np.meshgrid(*axes[::-1], indexing="ij")
    vertices = np.stack([g.ravel() for g in grids[::-1]], axis=-1)
    n_el = int(np.prod(nn))
    # element multi-index, direction 0 fastest
    pos = [np.arange(n_el) // int(np.prod(nn[:j])) % nn[j] for j in range(d)]
    vstride = [int(np.prod([n + 1 for n in nn[:j]])) for j in range(d)]
    estride = [int(np.prod(nn[:j])) for j in range(d)]
    base = sum(pos[j] * vstride[j] for j in range(d))
    elements = np.stack([base + sum(((v >> j) & 1) * vstride[j] for j in range(d))
                         for v in range(2 ** d)], axis=1)
    neighbors = -np.ones((n_el, d, 2), dtype=np.int64)
    own_id = np.arange(n_el)
    for axis in range(d):
        for side, step in ((0, -1), (1, 1)):
            q = pos[axis] + step
            if boundary_kind == "periodic":
                q = q % nn[axis]
            ok = (q >= 0) & (q < nn[axis])
            nbr = own_id + (q - pos[axis]) * estride[axis]
            neighbors[ok, axis, side] = nbr[ok]
    return OracleMesh(d, nn, vertices, elements, neighbors, boundary_kind)


def min_edge_length(mesh: OracleMesh) -> float:
    """Shortest straight element edge (reference mesh.py:294-304)."""
    x = mesh.vertices[mesh.elements]
    best = np.inf
    for j in range(mesh.d):
        lo = [v for v in range(2 ** mesh.d) if not (v >> j) & 1]
        hi = [v | (1 << j) for v in lo]
        best = min(best, float(np.linalg.norm(x[:, hi] - x[:, lo], axis=-1).min()))
    return best


def _tensor_apply(mats, arr, lead: int):
    """Contract tensor axes of ``arr`` (after ``lead`` batch axes, direction 0
    last) with one matrix per direction."""
    d = len(mats)
    out = arr
    for m, mat in enumerate(mats):
        ax = lead + (d - 1 - m)
        out = np.moveaxis(np.tensordot(out, mat, axes=([ax], [1])), -1, ax)
    return out


def geometry_nodes(mesh: OracleMesh, g: int,
                   mapping: Callable[[np.ndarray], np.ndarray] | None = None) -> np.ndarray:
    """Physical coordinates at the degree-g GL geometry nodes, shape
    (E, g+1, ..., g+1, d) with direction 0 on the last tensor axis.

    The straight element map is multilinear in the vertices; ``mapping``
    (optional) is then applied pointwise, giving the isoparametric
    interpolant of the composed map.
    """
    d = mesh.d
    xv = mesh.vertices[mesh.elements]          # (E, 2^d, d), vertex bit j = dir j
    xv = xv.reshape((mesh.n_elements,) + (2,) * d + (d,))  # dir 0 last tensor axis
    if g == 1 and mapping is None:
        return xv
    gl, _ = gauss_lobatto_rule(g + 1)
    lin = lagrange_matrix(np.array([0.0, 1.0]), gl)
    x = _tensor_apply([lin] * d, np.moveaxis(xv, -1, 1), lead=2)
    x = np.moveaxis(x, 1, -1)
    if mapping is not None:
        x = mapping(x)
    return x


def map_points(mesh: OracleMesh, pts, g: int = 1, mapping=None) -> np.ndarray:
    """Physical coordinates of a tensor point set per element (mesh.py:213-226)."""
    nodes = np.moveaxis(geometry_nodes(mesh, g, mapping), -1, 1)
    gl, _ = gauss_lobatto_rule(g + 1)
    val = lagrange_matrix(gl, np.asarray(pts, dtype=float))
    return np.moveaxis(_tensor_apply([val] * mesh.d, nodes, lead=2), 1, -1)


# The metric is evaluated in extended precision (np.longdouble: Lagrange
# rows, Jacobian sums, adjugate, determinant, normals) from the double nodal
# coordinates and rounded once.  The reference evaluates the same formulas in
# double with np.linalg.det / inv (mesh.py:249-252, 271-277); for its own
# (multilinear, g = 1) meshes the results agree to round-off (pinned by
# tests/test_oracle_golden.py).  For the degree-5 map of config 3 the double
# evaluation is only reproducible to ~1e-13: J ~ h is a sum of O(1)
# coordinates times derivative rows of size ~20, so the rounding of the rows
# (sum != 0) and the summation order both show up at |x| / h * 1e-16.  In
# extended precision the rows sum to zero at 1e-19 and the value no longer
# depends on the implementation (the device builder agrees to ~1 ulp).
LD = np.longdouble


def _jacobian(nodes_c: np.ndarray, g: int, pts_per_dir) -> np.ndarray:
    """J[e, i, m, ...points] = d x_i / d xi_m for GL-nodal coordinates
    (long double)."""
    d = nodes_c.shape[1]
    gl, _ = gauss_lobatto_rule(g + 1)
    val = [lagrange_matrix(gl, p, dtype=LD) for p in pts_per_dir]
    der = [lagrange_matrix(gl, p, "derivative", dtype=LD) for p in pts_per_dir]
    x = np.asarray(nodes_c).astype(LD)
    cols = []
    for m in range(d):
        mats = [der[j] if j == m else val[j] for j in range(d)]
        cols.append(_tensor_apply(mats, x, lead=2))
    return np.stack(cols, axis=2)


def _adjugate_det(jm):
    """adj[..., m, :] = det J * (J^{-T} e_m): in 3-D the cross product of the
    two other columns of J, in 2-D the rotated column; det = J[:, 0] . adj[0]."""
    d = jm.shape[-1]
    col = [jm[..., :, m] for m in range(d)]
    if d == 3:
        adj = np.stack([np.cross(col[1], col[2]), np.cross(col[2], col[0]),
                        np.cross(col[0], col[1])], axis=-2)
    else:
        adj = np.stack([np.stack([col[1][..., 1], -col[1][..., 0]], -1),
                        np.stack([-col[0][..., 1], col[0][..., 0]], -1)], axis=-2)
    det = np.sum(col[0] * adj[..., 0, :], axis=-1)
    return adj, det


def _volume(nodes_c, g, q):
    d = nodes_c.shape[1]
    pts, w = gauss_rule(q + 1)
    jac = _jacobian(nodes_c, g, [pts] * d)                  # (E, i, m, ...)
    jm = np.moveaxis(jac.reshape(jac.shape[:3] + (-1,)), 3, 1)  # (E, P, i, m)
    adj, det = _adjugate_det(jm)
    if np.any(det <= 0):
        raise ValueError("non-positive Jacobian determinant")
    inv = adj / det[..., None, None]                         # (E,P,m,i) = dxi_m/dx_i
    wt = w
    for _ in range(d - 1):
        wt = np.multiply.outer(w, wt)
    ext = (q + 1,) * d
    inv_jac = np.moveaxis(inv, 1, 3).reshape((nodes_c.shape[0], d, d) + ext)
    jxw = (det * wt.ravel()).reshape((nodes_c.shape[0],) + ext)
    return VolumeMetric(np.ascontiguousarray(inv_jac, dtype=np.float64),
                        jxw.astype(np.float64)), jm.astype(np.float64)


def _face(nodes_c, g, k, axis, side):
    d = nodes_c.shape[1]
    pts, w = gauss_rule(k + 1)
    per_dir = [pts if j != axis else np.array([float(side)]) for j in range(d)]
    jac = _jacobian(nodes_c, g, per_dir)
    jm = np.moveaxis(jac.reshape(jac.shape[:3] + (-1,)), 3, 1)
    adj, det = _adjugate_det(jm)
    if np.any(det <= 0):
        raise ValueError("non-positive Jacobian determinant on a face")
    nvec = (2 * side - 1) * adj[:, :, axis, :]               # det J^{-T} e_axis
    length = np.sqrt(np.sum(nvec * nvec, axis=-1))
    wt = np.ones(())
    for j in reversed(range(d)):
        if j != axis:
            wt = np.multiply.outer(wt, w)
    fext = (k + 1,) * (d - 1)
    e = nodes_c.shape[0]
    normal = np.moveaxis(nvec / length[..., None], 2, 1).reshape((e, d) + fext)
    return FaceMetric(np.ascontiguousarray(normal, dtype=np.float64),
                      (length * wt.ravel()).reshape((e,) + fext).astype(np.float64))


def _geometry_nodes_ld(mesh: OracleMesh, g: int, mapping) -> np.ndarray:
    """geometry_nodes evaluated in long double and not rounded (the metric's
    input: rounding coordinates ~1 to double would perturb J ~ h by 1e-13 h)."""
    d = mesh.d
    xv = mesh.vertices[mesh.elements].reshape((mesh.n_elements,) + (2,) * d + (d,))
    xv = xv.astype(LD)
    if g == 1 and mapping is None:
        return xv
    gl, _ = gauss_lobatto_rule(g + 1)
    lin = lagrange_matrix(np.array([0.0, 1.0]), gl, dtype=LD)
    x = np.moveaxis(_tensor_apply([lin] * d, np.moveaxis(xv, -1, 1), lead=2), 1, -1)
    return mapping(x) if mapping is not None else x


def precompute_geometry(mesh: OracleMesh, k: int, reduced_degrees=None,
                        g: int = 1, mapping=None) -> OracleGeometry:
    """Metric at degree-k Gauss points, reduced-degree cell point sets and the
    2d face groups (reference mesh.py:307-334)."""
    if reduced_degrees is None:
        reduced_degrees = tuple(range(k - 2, -1, -2))
    nodes = _geometry_nodes_ld(mesh, g, mapping)
    nodes_c = np.moveaxis(nodes, -1, 1)                      # (E, d, ...)
    vol = {}
    vol[k], jm = _volume(nodes_c, g, k)
    scale = np.max(np.abs(jm))
    dev = np.abs(jm - jm[:, :1]).max(axis=(1, 2, 3))
    off = np.abs(jm * (1.0 - np.eye(mesh.d))).max(axis=(1, 2, 3))
    cart = (dev < 1e-12 * scale) & (off < 1e-12 * scale)
    for q in sorted(set(int(v) for v in reduced_degrees) - {k}):
        if not 0 <= q <= k:
            raise ValueError(f"reduced degree {q} outside 0..{k}")
        vol[q], _ = _volume(nodes_c, g, q)
    face = {(a, s): _face(nodes_c, g, k, a, s) for a in range(mesh.d) for s in (0, 1)}
    return OracleGeometry(k, vol, face, min_edge_length(mesh), cart)
