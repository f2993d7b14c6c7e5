"""Host-side mesh, material and geometry setup (the hot path's input contract).

Mirrors the data the reference operator reads:
``Mesh.neighbors`` / element order (``/root/reference/pkg/src/wavekernel/
mesh.py:69-127``), ``Material`` (mesh.py:145-159) and the
``GeometryCache`` layout (mesh.py:162-188).  Reference objects are accepted
unchanged by :class:`~paper_1805_03981_b200.operator.AcousticOperator`;
the builders here exist so the GPU path runs where the reference is not
installed (the GPU box) and at sizes the reference's dense per-point geometry
cannot reach (config 5 would need ~15 GB of host metric arrays).

* :func:`affine_geometry` derives the per-element constant Jacobian of affine
  cells directly from the vertices (no per-point arrays).
* :func:`precompute_geometry` builds the full per-point metric for curved
  isoparametric maps of geometry degree ``g`` (BASELINE config 3); with
  ``device="cuda"`` the metric is evaluated by the ``wk_curved_metric``
  kernel from the nodal coordinates and the arrays stay on the GPU
  (config 3 setup 13 s -> well under a second).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import rules


class GeometryError(ValueError):
    """Inverted or degenerate element map (reference mesh.py:20-21)."""


@dataclass(frozen=True)
class Mesh:
    d: int
    n_per_dim: tuple
    vertices: np.ndarray
    elements: np.ndarray
    neighbors: np.ndarray
    boundary_kind: str

    @property
    def n_elements(self) -> int:
        return self.elements.shape[0]

    @property
    def periodic(self) -> bool:
        return self.boundary_kind == "periodic"


@dataclass(frozen=True)
class Material:
    c: np.ndarray
    rho: np.ndarray

    def __post_init__(self):
        if np.any(np.asarray(self.c) <= 0) or np.any(np.asarray(self.rho) <= 0):
            raise ValueError("material constants must be positive")

    @classmethod
    def uniform(cls, mesh, c: float = 1.0, rho: float = 1.0):
        e = mesh.n_elements
        return cls(c=np.full(e, float(c)), rho=np.full(e, float(rho)))


def build_cartesian(n_per_dim, d: int, boundary_kind: str = "sound_soft") -> Mesh:
    """Uniform mesh of [0,1]^d, element e = i0 + n0 (i1 + n1 i2)."""
    if d not in (2, 3):
        raise ValueError("dimension must be 2 or 3")
    if boundary_kind not in ("sound_soft", "periodic"):
        raise ValueError(f"unknown boundary kind {boundary_kind!r}")
    nn = (int(n_per_dim),) * d if np.isscalar(n_per_dim) else tuple(int(v) for v in n_per_dim)
    if len(nn) != d or min(nn) < 1:
        raise ValueError("bad element counts")
    nv = [n + 1 for n in nn]
    vid = np.arange(int(np.prod(nv)))
    vertices = np.stack([np.linspace(0.0, 1.0, nv[j])[(vid // int(np.prod(nv[:j]))) % nv[j]]
                         for j in range(d)], axis=-1)
    n_el = int(np.prod(nn))
    eid = np.arange(n_el)
    pos = [(eid // int(np.prod(nn[:j]))) % nn[j] for j in range(d)]
    vbase = sum(pos[j] * int(np.prod(nv[:j])) for j in range(d))
    elements = np.empty((n_el, 2 ** d), dtype=np.int64)
    for v in range(2 ** d):
        elements[:, v] = vbase + sum(((v >> j) & 1) * int(np.prod(nv[:j])) for j in range(d))
    neighbors = np.full((n_el, d, 2), -1, dtype=np.int64)
    for j in range(d):
        stride = int(np.prod(nn[:j]))
        for side, step in ((0, -1), (1, 1)):
            q = pos[j] + step
            if boundary_kind == "periodic":
                q %= nn[j]
            ok = (q >= 0) & (q < nn[j])
            neighbors[ok, j, side] = (eid + (q - pos[j]) * stride)[ok]
    return Mesh(d, nn, vertices, elements, neighbors, boundary_kind)


def map_vertices(mesh: Mesh, mapping: Callable[[np.ndarray], np.ndarray]) -> Mesh:
    """Apply a pointwise map to the vertex coordinates (for h_min and the
    straight-edge Courant length of curved meshes)."""
    return Mesh(mesh.d, mesh.n_per_dim, mapping(mesh.vertices), mesh.elements,
                mesh.neighbors, mesh.boundary_kind)


def deform(mesh: Mesh, amplitude: float) -> Mesh:
    """Move every vertex by amplitude * prod_j sin(pi x_j) in each coordinate
    (reference mesh.py:129-142): zero on the cube's boundary, so periodic
    identification survives; the cells become multilinear (per-point metric)."""
    if amplitude < 0 or amplitude >= 0.5 / max(mesh.n_per_dim):
        raise ValueError("amplitude outside the inversion-safe range")
    shift = amplitude * np.sin(np.pi * mesh.vertices).prod(axis=1)
    return map_vertices(mesh, lambda x: x + shift[:, None])


def min_edge_length(mesh) -> float:
    """Shortest straight element edge (reference mesh.py:294-304)."""
    x = mesh.vertices[mesh.elements]
    best = np.inf
    for j in range(mesh.d):
        for v in range(2 ** mesh.d):
            if (v >> j) & 1:
                continue
            best = min(best, float(np.linalg.norm(x[:, v | (1 << j)] - x[:, v], axis=1).min()))
    return best


# ---------------------------------------------------------------------------
# affine cells: per-element constant metric


@dataclass(frozen=True)
class AffineGeometry:
    """Constant metric of affine cells (no per-point arrays).

    G[e, m, i] = d xi_m / d x_i, det[e] = det J, normal[e, m, s, :] outward
    unit normal of face (m, s), fscale[e, m, s] = face JxW / (w x w) / det J.
    """
    degree: int
    G: np.ndarray
    det: np.ndarray
    normal: np.ndarray
    fscale: np.ndarray
    h_min: float
    cartesian_flag: np.ndarray = field(repr=False)


def affine_geometry(mesh, k: int, tol: float = 1e-12) -> AffineGeometry:
    """Derive the constant Jacobian of every cell from its 2^d vertices.

    Raises ValueError when a cell is not affine (use precompute_geometry).
    """
    d = mesh.d
    x = mesh.vertices[mesh.elements]                 # (E, 2^d, d)
    J = np.stack([x[:, 1 << m] - x[:, 0] for m in range(d)], axis=2)  # J[e, i, m]
    pred = x[:, :1] + np.stack(
        [sum(((v >> m) & 1) * J[:, :, m] for m in range(d)) for v in range(2 ** d)], axis=1)
    scale = max(np.max(np.abs(x)), 1.0)
    if np.max(np.abs(pred - x)) > tol * scale:
        raise ValueError("mesh has non-affine cells; build per-point geometry")
    det = np.linalg.det(J)
    if np.any(det <= 0):
        raise GeometryError("non-positive Jacobian determinant")
    G = np.linalg.inv(J)                              # G[e, m, i] = d xi_m / d x_i
    normal = np.empty((mesh.n_elements, d, 2, d))
    fscale = np.empty((mesh.n_elements, d, 2))
    for m in range(d):
        row = det[:, None] * G[:, m, :]
        length = np.linalg.norm(row, axis=1)
        for s in (0, 1):
            normal[:, m, s, :] = (2.0 * s - 1.0) * row / length[:, None]
            fscale[:, m, s] = length / det
    off = np.abs(J * (1.0 - np.eye(d))).max(axis=(1, 2))
    cart = off < tol * np.abs(J).max(axis=(1, 2))
    # uniform grids: the per-element vertex differences agree to round-off
    # (non-dyadic spacings differ in the last bit).  Canonicalise to element
    # 0's record so every element -- and every slab of a partitioned mesh --
    # sees bit-identical constants (one geometry class, bitwise multi-GPU
    # reproducibility).  The change is below 1e-15 relative.
    rec = np.concatenate([G.reshape(len(G), -1), det[:, None]], axis=1)
    scale = np.maximum(np.abs(rec).max(axis=0), 1e-300)
    if np.max(np.abs(rec - rec[:1]) / scale) < 1e-13:
        G = np.broadcast_to(G[:1], G.shape).copy()
        det = np.broadcast_to(det[:1], det.shape).copy()
        normal = np.broadcast_to(normal[:1], normal.shape).copy()
        fscale = np.broadcast_to(fscale[:1], fscale.shape).copy()
    return AffineGeometry(k, G, det, normal, fscale, min_edge_length(mesh), cart)


# ---------------------------------------------------------------------------
# curved cells: per-point metric in the reference GeometryCache layout


@dataclass(frozen=True)
class VolumeGeometry:
    inv_jac: np.ndarray
    jxw: np.ndarray


@dataclass(frozen=True)
class FaceGeometry:
    normal: np.ndarray
    jxw: np.ndarray


@dataclass(frozen=True)
class GeometryCache:
    degree: int
    vol: dict
    face: dict
    h_min: float
    cartesian_flag: np.ndarray = field(repr=False)


def lagrange(nodes, pts, derivative: bool = False) -> np.ndarray:
    """mat[i, j] = L_j(pts_i) (or L_j') for the Lagrange basis on ``nodes``
    (the product formula, double)."""
    nodes = np.asarray(nodes, dtype=float)
    pts = np.asarray(pts, dtype=float)
    n = nodes.size
    out = np.zeros((pts.size, n))
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


def _contract(mats, arr, lead):
    d = len(mats)
    for m, mat in enumerate(mats):
        ax = lead + d - 1 - m
        arr = np.moveaxis(np.tensordot(arr, mat, axes=([ax], [1])), -1, ax)
    return arr


def _gl(g: int) -> np.ndarray:
    return np.array([0.0, 1.0]) if g == 1 else rules.gl_points(g)


def geometry_nodes(mesh, g: int, mapping=None) -> np.ndarray:
    """(E, d, g+1, ..., g+1) physical coordinates at the degree-g GL nodes of
    the straight map, optionally composed with a pointwise ``mapping``."""
    d = mesh.d
    xv = mesh.vertices[mesh.elements].reshape((mesh.n_elements,) + (2,) * d + (d,))
    xv = np.moveaxis(xv, -1, 1)
    if g == 1 and mapping is None:
        return xv
    lin = lagrange([0.0, 1.0], _gl(g))
    x = _contract([lin] * d, xv, 2)
    if mapping is not None:
        x = np.moveaxis(mapping(np.moveaxis(x, 1, -1)), -1, 1)
    return x


def geometry_nodes_ld(mesh, g: int, mapping=None) -> np.ndarray:
    """geometry_nodes in long double (the metric builders' input): the
    straight map and ``mapping`` are evaluated in extended precision and NOT
    rounded, so the metric is a smooth function of the GL points (rounding
    the coordinates to double would perturb J ~ h by ~|x| ulp ~ 1e-13 h)."""
    d = mesh.d
    xv = mesh.vertices[mesh.elements].reshape((mesh.n_elements,) + (2,) * d + (d,))
    xv = np.moveaxis(xv, -1, 1).astype(rules.LD)
    if g == 1 and mapping is None:
        return xv
    x = _contract([rules.lagrange_ld([0.0, 1.0], _gl(g))] * d, xv, 2)
    if mapping is not None:
        x = np.moveaxis(mapping(np.moveaxis(x, 1, -1)), -1, 1)
    return x


def map_points(mesh, pts, g: int = 1, mapping=None) -> np.ndarray:
    """Physical coordinates (E, n, ..., n, d) of a tensor reference point set."""
    nodes = geometry_nodes(mesh, g, mapping)
    val = lagrange(_gl(g), pts)
    return np.moveaxis(_contract([val] * mesh.d, nodes, 2), 1, -1)


def _cofactor_inverse(Jm):
    """det, inverse and cofactor matrix of (..., d, d) matrices, in the dtype
    of ``Jm`` (inv[..., m, i] = d xi_m / d x_i = cof[..., i, m] / det)."""
    d = Jm.shape[-1]
    J = lambda i, m: Jm[..., i, m]
    cof = np.empty(Jm.shape, dtype=Jm.dtype)
    if d == 2:
        cof[..., 0, 0], cof[..., 0, 1] = J(1, 1), -J(1, 0)
        cof[..., 1, 0], cof[..., 1, 1] = -J(0, 1), J(0, 0)
        det = J(0, 0) * J(1, 1) - J(0, 1) * J(1, 0)
    else:
        for i in range(3):
            for m in range(3):
                i1, i2 = (i + 1) % 3, (i + 2) % 3
                m1, m2 = (m + 1) % 3, (m + 2) % 3
                cof[..., i, m] = J(i1, m1) * J(i2, m2) - J(i1, m2) * J(i2, m1)
        det = J(0, 0) * cof[..., 0, 0] + J(0, 1) * cof[..., 0, 1] + J(0, 2) * cof[..., 0, 2]
    inv = np.swapaxes(cof, -1, -2) / det[..., None, None]
    return det, inv, cof


def _metric(nodes, g, per_dir):
    """Jacobian (E, P, i, m), det, inverse and cofactors at a tensor point
    set, evaluated in long double from the long-double nodal coordinates with
    long-double Lagrange rows: the derivative rows then sum to zero far below
    double round-off, so J ~ h is not polluted by |x| ~ 1 (SURVEY.md §8c
    item 1).  The caller rounds once.  The device builder (wk_curved_metric)
    does the same in double-double; the two agree to ~1 ulp
    (tests/test_gpu_geometry.py)."""
    d = nodes.shape[1]
    gl = _gl(g)
    val = [rules.lagrange_ld(gl, p) for p in per_dir]
    der = [rules.lagrange_ld(gl, p, True) for p in per_dir]
    x = np.asarray(nodes, dtype=rules.LD)
    J = np.stack([_contract([der[j] if j == m else val[j] for j in range(d)], x, 2)
                  for m in range(d)], axis=2)          # (E, i, m, pts...)
    E = nodes.shape[0]
    Jm = np.moveaxis(J.reshape(E, d, d, -1), 3, 1)     # (E, P, i, m)
    det, inv, cof = _cofactor_inverse(Jm)
    if np.any(det <= 0):
        raise GeometryError("non-positive Jacobian determinant")
    return Jm, det, inv, cof


def precompute_geometry(mesh, k: int, reduced_degrees=None, g: int = 1,
                        mapping=None, device=None) -> GeometryCache:
    """Per-point metric at the degree-k (and reduced) Gauss points plus the 2d
    face groups, in the reference GeometryCache layout (mesh.py:245-334):
    ``inv_jac = J^{-1}``, ``jxw = det J * w``, face normal
    ``(2s-1) det J^{-T} e_m / |.|`` and face ``jxw = |det J^{-T} e_m| * w``
    (mesh.py:249-286; ``det J^{-T} e_m`` is column m of the cofactor matrix).

    ``device`` (e.g. ``"cuda"``): evaluate on the GPU; the arrays are then
    CUDA tensors in the same layout (the operator consumes them in place)."""
    if reduced_degrees is None:
        reduced_degrees = tuple(range(k - 2, -1, -2))
    if device is not None:
        return _device_geometry(mesh, k, reduced_degrees, g, mapping, device)
    d, E = mesh.d, mesh.n_elements
    nodes = geometry_nodes_ld(mesh, g, mapping)
    chunk = max(1, 1 << 20 // max(1, (k + 1) ** d * d * d))
    parts = [slice(a, min(E, a + chunk)) for a in range(0, E, chunk)]
    vol = {}
    cart = None
    for q in [k] + sorted(set(int(v) for v in reduced_degrees) - {k}):
        pts, w = rules.gauss_points(q), rules.gauss_weights(q)
        wt = w
        for _ in range(d - 1):
            wt = np.multiply.outer(w, wt)
        ext = (q + 1,) * d
        inv_jac = np.empty((E, d, d) + ext)
        jxw = np.empty((E,) + ext)
        stats = np.empty((E, 3))
        for sl in parts:
            Jm, det, inv, _ = _metric(nodes[sl], g, [pts] * d)
            n_e = Jm.shape[0]
            inv_jac[sl] = np.moveaxis(inv, 1, 3).reshape((n_e, d, d) + ext)
            jxw[sl] = (det * wt.ravel()).reshape((n_e,) + ext)
            Jd = Jm.astype(np.float64)
            stats[sl, 0] = np.abs(Jd - Jd[:, :1]).max(axis=(1, 2, 3))
            stats[sl, 1] = np.abs(Jd * (1.0 - np.eye(d))).max(axis=(1, 2, 3))
            stats[sl, 2] = np.abs(Jd).max(axis=(1, 2, 3))
        vol[q] = VolumeGeometry(inv_jac, jxw)
        if q == k:
            scale = stats[:, 2].max() if E else 0.0
            cart = (stats[:, 0] < 1e-12 * scale) & (stats[:, 1] < 1e-12 * scale)
    pts, w = rules.gauss_points(k), rules.gauss_weights(k)
    fext = (k + 1,) * (d - 1)
    face = {}
    for m in range(d):
        wt = np.ones(())
        for j in reversed(range(d)):
            if j != m:
                wt = np.multiply.outer(wt, w)
        for s in (0, 1):
            per_dir = [pts if j != m else np.array([float(s)]) for j in range(d)]
            normal = np.empty((E, d) + fext)
            fjxw = np.empty((E,) + fext)
            for sl in parts:
                _, _, _, cof = _metric(nodes[sl], g, per_dir)
                nvec = (2 * s - 1) * cof[:, :, :, m]          # (e, P, i)
                length = np.sqrt(np.sum(nvec * nvec, axis=-1))
                n_e = nvec.shape[0]
                normal[sl] = np.moveaxis(nvec / length[..., None], 2, 1).reshape((n_e, d) + fext)
                fjxw[sl] = (length * wt.ravel()).reshape((n_e,) + fext)
            face[(m, s)] = FaceGeometry(normal, fjxw)
    return GeometryCache(k, vol, face, min_edge_length(mesh), cart)


def _dd_split(t: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """long double -> (hi, lo) doubles with hi + lo = t to 64 bits."""
    hi = t.astype(np.float64)
    lo = (t - hi.astype(rules.LD)).astype(np.float64)
    return np.ascontiguousarray(hi.ravel()), np.ascontiguousarray(lo.ravel())


def _device_geometry(mesh, k, reduced_degrees, g, mapping, device) -> GeometryCache:
    """precompute_geometry on the GPU (wk_curved_metric, csrc/wk_geometry.cu).

    The nodal coordinates of the map are built on the host (the mapping is a
    Python callable); the per-point metric, which is what costs, is evaluated
    by the kernel in double-double from long-double Lagrange rows (passed as
    hi/lo pairs), the same arithmetic as the host builder above.
    cartesian_flag follows the reference's rule from the per-element Jacobian
    statistics the volume pass returns."""
    import ctypes
    import torch
    from ._lib import check, dptr, lib
    d, E = mesh.d, mesh.n_elements
    dev = torch.device(device)
    # nodal coordinates as double-double (hi, lo) pairs of the long-double map
    nodes_ld = geometry_nodes_ld(mesh, g, mapping)
    n_hi = nodes_ld.astype(np.float64)
    n_lo = (nodes_ld - n_hi.astype(rules.LD)).astype(np.float64)
    del nodes_ld
    nodes = torch.from_numpy(np.ascontiguousarray(np.stack([n_hi, n_lo]))).to(dev)
    del n_hi, n_lo
    gl = _gl(g)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None

    def run(per_dir, wts, face=(-1, 0), stats=None):
        npts = np.array([len(p) for p in per_dir], dtype=np.int32)
        val = _dd_split(np.concatenate([rules.lagrange_ld(gl, p).ravel() for p in per_dir]))
        der = _dd_split(np.concatenate([rules.lagrange_ld(gl, p, True).ravel()
                                        for p in per_dir]))
        wts = np.ascontiguousarray(np.ravel(wts), dtype=np.float64)
        npt = int(np.prod(npts))
        jxw = torch.empty((E, npt), dtype=torch.float64, device=dev)
        if face[0] < 0:
            inv = torch.empty((E, d, d, npt), dtype=torch.float64, device=dev)
            nrm = None
        else:
            inv = None
            nrm = torch.empty((E, d, npt), dtype=torch.float64, device=dev)
        check(lib().wk_curved_metric(d, g, E, P(nodes), dptr(npts), dptr(val[0]), dptr(val[1]),
                                     dptr(der[0]), dptr(der[1]), dptr(wts), face[0], face[1],
                                     P(inv), P(jxw), P(nrm), P(stats), P(bad), stream))
        return inv, jxw, nrm

    vol = {}
    cart = None
    for q in [k] + sorted(set(int(v) for v in reduced_degrees) - {k}):
        pts, w = rules.gauss_points(q), rules.gauss_weights(q)
        wt = w
        for _ in range(d - 1):
            wt = np.multiply.outer(w, wt)
        stats = torch.empty((E, 3), dtype=torch.float64, device=dev) if q == k else None
        inv, jxw, _ = run([pts] * d, wt, stats=stats)
        ext = (q + 1,) * d
        vol[q] = VolumeGeometry(inv.reshape((E, d, d) + ext), jxw.reshape((E,) + ext))
        if q == k:
            st = stats.cpu().numpy()
            scale = float(st[:, 2].max()) if E else 0.0
            cart = (st[:, 0] < 1e-12 * scale) & (st[:, 1] < 1e-12 * scale)
    pts, w = rules.gauss_points(k), rules.gauss_weights(k)
    face = {}
    for m in range(d):
        for s in (0, 1):
            per_dir = [pts if j != m else np.array([float(s)]) for j in range(d)]
            wt = np.ones(())
            for j in reversed(range(d)):
                if j != m:
                    wt = np.multiply.outer(wt, w)
            _, jxw, nrm = run(per_dir, wt, face=(m, s))
            fext = (k + 1,) * (d - 1)
            face[(m, s)] = FaceGeometry(nrm.reshape((E, d) + fext), jxw.reshape((E,) + fext))
    if int(bad.item()) != 0:
        raise GeometryError("non-positive Jacobian determinant")
    return GeometryCache(k, vol, face, min_edge_length(mesh), cart)
