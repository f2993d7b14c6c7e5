"""GPU drop-in for the reference ``AcousticOperator``.

Mirrors ``/root/reference/pkg/src/wavekernel/operator.py``: same constructor
``AcousticOperator(mesh, geometry, material, flux=FluxParams(), counter=None)``
(:93-123), same attributes (``mesh, geometry, material, flux, k, d, n_comp,
gl_to_g, g_to_gl, _d_co``), same methods (``apply_K`` :149, ``_check``
:127, ``apply_inverse_mass`` :250, ``apply_mass`` :260, ``rhs`` :268,
``to_gauss_values`` :276, ``from_gauss_weighted`` :279, ``apply_local_S``
:286, ``resize_values`` :308) and the same ``ValueError`` contract.

Every method runs hand-written sm_100a CUDA through the C ABI
(``include/wavekernel_b200.h``); there is no CPU path.  ``StateVector.data``
may be a numpy array (copied to the GPU and back, as a drop-in for the
reference's numpy states) or a CUDA ``torch.Tensor`` (stays on the device;
what the steppers use).  PyTorch is only the owner of device memory and the
current stream.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, cost
from ._lib import check, dptr, lib
from .mesh import AffineGeometry, affine_geometry


def _torch():
    import torch
    return torch


@dataclass
class StateVector:
    """Element-contiguous coefficients (E, d+1, n, ..., n), reference layout
    (operator.py:33-55).  ``data`` is a numpy array or a CUDA torch tensor."""
    data: object
    degree: int
    dim: int
    basis: str = "gl"

    def copy(self) -> "StateVector":
        d = self.data.clone() if not isinstance(self.data, np.ndarray) else self.data.copy()
        return StateVector(d, self.degree, self.dim, self.basis)

    @classmethod
    def zeros(cls, n_elements: int, degree: int, dim: int, device=None) -> "StateVector":
        shape = (n_elements, dim + 1) + (degree + 1,) * dim
        if device is None:
            return cls(np.zeros(shape), degree, dim)
        torch = _torch()
        return cls(torch.zeros(shape, dtype=torch.float64, device=device), degree, dim)

    def numpy(self) -> np.ndarray:
        if isinstance(self.data, np.ndarray):
            return self.data
        return self.data.detach().cpu().numpy()


@dataclass(frozen=True)
class FluxParams:
    """HDG stabilization (operator.py:58-67): tau defaults to 1/(c rho)."""
    tau: float | None = None
    stabilization: bool = True


class _Table:
    """Host view of a 1-D table with the reference BasisMatrix1D ``.matrix``."""

    def __init__(self, matrix, nodes=None):
        self.matrix = matrix
        self.nodes = nodes

    @property
    def shape(self):
        return self.matrix.shape


def _is_tensor(x) -> bool:
    return hasattr(x, "data_ptr") and hasattr(x, "is_cuda")


def _contig(x):
    """FP64 contiguous host array or CUDA tensor (device geometry)."""
    if _is_tensor(x):
        return x.to(dtype=_torch().float64).contiguous()
    return np.ascontiguousarray(x, dtype=np.float64)


def _any_ptr(x):
    if _is_tensor(x):
        return ctypes.cast(ctypes.c_void_p(x.data_ptr()), ctypes.POINTER(ctypes.c_double))
    return dptr(x)


def _host_geometry(geo):
    from .mesh import FaceGeometry, GeometryCache, VolumeGeometry
    h = lambda x: x.cpu().numpy() if _is_tensor(x) else np.asarray(x)
    return GeometryCache(geo.degree,
                         {q: VolumeGeometry(h(v.inv_jac), h(v.jxw)) for q, v in geo.vol.items()},
                         {f: FaceGeometry(h(v.normal), h(v.jxw)) for f, v in geo.face.items()},
                         geo.h_min, np.asarray(geo.cartesian_flag))


def hdg_flux(minus, plus, n, c, rho, tau):
    """Numerical trace flux directed outward from the minus side
    (reference operator.py:70-87): ``minus``/``plus`` are (v, p) with the d
    velocity components along the leading axis, ``n`` the minus side's unit
    normal; tau None or 0 leaves the central flux.  The fused kernels inline
    the split-form variant of this flux; this pointwise form is
    the reference's test-facing API.  Works on numpy arrays or torch tensors."""
    v_m, p_m = minus
    v_p, p_p = plus
    tau = 0.0 if tau is None else float(tau)
    vn_m = (n * v_m).sum(axis=0) if isinstance(v_m, np.ndarray) else (n * v_m).sum(0)
    vn_p = (n * v_p).sum(axis=0) if isinstance(v_p, np.ndarray) else (n * v_p).sum(0)
    flux_v = (p_m + p_p) / (2.0 * rho) * n
    flux_p = 0.5 * c ** 2 * rho * (vn_m + vn_p)
    if tau != 0.0:
        flux_v = flux_v + (vn_m - vn_p) / (2.0 * rho * tau) * n
        flux_p = flux_p + 0.5 * c ** 2 * rho * tau * (p_m - p_p)
    return flux_v, flux_p


class AcousticOperator:
    """Sum-factorized K, M^{-1}, M and local S on the GPU (see module doc)."""

    def __init__(self, mesh, geometry, material, flux: FluxParams = FluxParams(),
                 counter=None, device: str = "cuda", n_ghost_faces: int = 0):
        torch = _torch()
        if geometry is None:
            raise ValueError("geometry is required (use mesh.affine_geometry for large "
                             "affine meshes)")
        if np.asarray(geometry.cartesian_flag).shape[0] != mesh.n_elements:
            raise ValueError("geometry was built for a different mesh")
        self.mesh = mesh
        self.geometry = geometry
        self.material = material
        self.flux = flux
        from .cost import KernelCounter
        self.counter = counter if counter is not None else KernelCounter()
        self.k = int(geometry.degree)
        self.d = int(mesh.d)
        self.n_comp = self.d + 1
        if not 1 <= self.k <= 8:
            raise ValueError("GPU operator supports degrees 1..8")
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise RuntimeError("AcousticOperator runs on CUDA only (no CPU fallback)")
        k = self.k
        self.gl_to_g = _Table(_lib.basis_table("gl_to_g", k), _lib.basis_table("gl_points", k))
        self.g_to_gl = _Table(_lib.basis_table("g_to_gl", k))
        self._d_co = {q: _Table(_lib.basis_table("d_co", q)) for q in self._degrees()}
        E = mesh.n_elements
        rho = np.asarray(material.rho, dtype=np.float64)
        c = np.asarray(material.c, dtype=np.float64)
        self.inv_rho = 1.0 / rho
        self.c2rho = c ** 2 * rho
        tau = 1.0 / (c * rho) if flux.tau is None else np.full(E, float(flux.tau))
        if np.any(tau <= 0):
            raise ValueError("stabilization must be positive")
        self.tau = tau
        self._n_ghost = int(n_ghost_faces)
        self._ctx = ctypes.c_void_p()
        self._keep = []
        self._build_ctx(np.ascontiguousarray(tau, dtype=np.float64))

    # -- context ----------------------------------------------------------
    def _degrees(self):
        if isinstance(self.geometry, AffineGeometry) or not hasattr(self.geometry, "vol"):
            return tuple(range(self.k + 1))
        return tuple(sorted(self.geometry.vol))

    def _build_ctx(self, tau):
        d, k, E = self.d, self.k, self.mesh.n_elements
        keep = self._keep
        desc = _lib.WkDesc()
        desc.dim, desc.degree, desc.n_elements = d, k, E
        desc.n_ghost_faces = int(getattr(self, "_n_ghost", 0))
        nbr = np.ascontiguousarray(self.mesh.neighbors, dtype=np.int32)
        ir = np.ascontiguousarray(self.inv_rho)
        c2r = np.ascontiguousarray(self.c2rho)
        keep += [nbr, ir, c2r, tau]
        desc.neighbors, desc.inv_rho, desc.c2rho, desc.tau = dptr(nbr), dptr(ir), dptr(c2r), dptr(tau)
        desc.stabilization = 1 if self.flux.stabilization else 0
        aff = self._affine_view()
        if aff is not None:
            G, det, normal, fscale = aff
            rec = np.concatenate([G.reshape(E, -1), normal.reshape(E, -1),
                                  fscale.reshape(E, -1), det.reshape(E, 1)], axis=1)
            # uniform meshes: element records agree to round-off (vertex
            # differences of non-dyadic spacings differ in the last bit); use
            # one class so the single-class fast kernels apply
            scale = np.maximum(np.max(np.abs(rec), axis=0), 1e-300)
            if np.max(np.abs(rec - rec[:1]) / scale) < 1e-13:
                uniq, inv = rec[:1], np.zeros(E, dtype=np.int64)
            else:
                uniq, inv = np.unique(rec, axis=0, return_inverse=True)
            nc = uniq.shape[0]
            off = [0, d * d, 3 * d * d, 3 * d * d + 2 * d]
            cG = np.ascontiguousarray(uniq[:, off[0]:off[1]])
            cN = np.ascontiguousarray(uniq[:, off[1]:off[2]])
            cF = np.ascontiguousarray(uniq[:, off[2]:off[3]])
            cD = np.ascontiguousarray(uniq[:, off[3]])
            cls = np.ascontiguousarray(inv.reshape(-1), dtype=np.int32)
            keep += [cG, cN, cF, cD, cls]
            desc.geometry_mode = _lib.WK_GEOM_AFFINE
            desc.n_classes = nc
            desc.geo_class = dptr(cls) if nc > 1 else None
            desc.affine_G, desc.affine_det = dptr(cG), dptr(cD)
            desc.affine_normal, desc.affine_fscale = dptr(cN), dptr(cF)
            self.geometry_mode = "affine"
            self.n_geometry_classes = nc
        else:
            geo = self.geometry
            degs = [k] + sorted(q for q in geo.vol if q != k)
            ij = [_contig(geo.vol[q].inv_jac) for q in degs]
            jw = [_contig(geo.vol[q].jxw) for q in degs]
            fn = [_contig(geo.face[(m, s)].normal) for m in range(d) for s in (0, 1)]
            fj = [_contig(geo.face[(m, s)].jxw) for m in range(d) for s in (0, 1)]
            dg = np.array(degs, dtype=np.int32)
            P = ctypes.POINTER(ctypes.c_double)
            arr = lambda xs: (P * len(xs))(*[_any_ptr(x) for x in xs])
            pij, pjw, pfn, pfj = arr(ij), arr(jw), arr(fn), arr(fj)
            keep += [ij, jw, fn, fj, dg, pij, pjw, pfn, pfj]
            desc.geometry_mode = _lib.WK_GEOM_CURVED
            desc.n_classes = 0
            desc.n_curved_degrees = len(degs)
            desc.curved_degrees = dptr(dg)
            desc.curved_inv_jac, desc.curved_jxw = pij, pjw
            desc.face_normal, desc.face_jxw = pfn, pfj
            self.geometry_mode = "curved"
            self.n_geometry_classes = E
        check(lib().wk_ctx_create(ctypes.byref(desc), ctypes.byref(self._ctx)))
        self._keep = []  # the library copied everything it needs
        self.tile_order = self._structured_order()
        if self.tile_order is not None:
            check(lib().wk_set_tile_order(self._ctx, *self.tile_order))
        # small Cartesian meshes (config 1): whole LSRK runs in one cluster
        # launch (wk_lsrk_run, csrc/wk_small.cuh); WK_SMALL=0 disables
        import os
        self.small_run = os.environ.get("WK_SMALL", "1") != "0" and \
            bool(lib().wk_lsrk_run_supported(self._ctx))

    # L2 traffic per element of one LSRK stage: read u, r; write u, r
    _STAGE_STREAMS = 4

    def _structured_order(self):
        """(chunk, n_slow, n_blocks) for wk_set_tile_order, or None.

        On an x-fastest structured 3-D mesh (reference numbering e = i0 + n0
        (i1 + n1 i2), mesh.py:88-89) the persistent kernels stream whole
        z-layers between an element and its z-neighbours; once a layer's
        traffic exceeds what L2 keeps, the neighbours' face values are
        re-read from DRAM (config 5: 1.17x the algorithmic reads).  Chunks of
        ``by`` y-rows visited block-major keep both z-neighbours within one
        chunk (<= 40 MB of traffic) of the element.  WK_TILE_ORDER=0 disables.

        Config 5, sustained (tools/sustain.py), 2 / 4 / 8 / 16 / 32 rows:
        15.3 / 14.85 / 14.60 / 14.48 / 14.88 ms/step.  Before the streamed
        vectors carried the L2 evict_first hint (wk_common.cuh) 16 rows were
        METASTABLE: on some boards the run dropped, at random, into the state
        where the z-faces miss L2 (18.8 ms/step, the mesh-order number) and
        stayed there; with the hint even mesh order holds 15.8."""
        import os
        if os.environ.get("WK_TILE_ORDER", "1") == "0" or self.d != 3 or self._n_ghost:
            return None
        # measured: config 5 (k = 4) reads 9.81 -> 8.90 GB per stage and runs
        # 1 % faster; config 4 (k = 7) is 1 % slower, so large k keeps mesh order
        if self.k > 5 and os.environ.get("WK_TILE_ORDER") != "1":
            return None
        nn = getattr(self.mesh, "n_per_dim", None)
        if nn is None or np.ndim(nn) == 0 or len(nn) != 3:
            return None
        nx, ny, nz = (int(v) for v in nn)
        E = self.mesh.n_elements
        if nx * ny * nz != E or E >= 2 ** 32:
            return None
        per = self._STAGE_STREAMS * self.n_comp * (self.k + 1) ** 3 * 8
        if nx * ny * per <= 48e6:
            return None
        by = max([b for b in range(1, ny + 1) if ny % b == 0 and nx * b * per <= 40e6] or [1])
        if os.environ.get("WK_TILE_BY"):          # chunk-size experiments
            by = int(os.environ["WK_TILE_BY"])
            if by < 1 or ny % by:
                return None
        if by == ny:
            return None
        # the numbering must be the structured one: +x, +y, +z neighbours
        nbr = np.asarray(self.mesh.neighbors)
        e = np.arange(E)
        i0, i1, i2 = e % nx, (e // nx) % ny, e // (nx * ny)
        for axis, (pos, n, stride) in enumerate(((i0, nx, 1), (i1, ny, nx), (i2, nz, nx * ny))):
            inner = pos < n - 1
            if not np.array_equal(nbr[inner, axis, 1], e[inner] + stride):
                return None
        return nx * by, nz, ny // by

    def _affine_view(self, rtol: float = 1e-12):
        """(G, det, normal, fscale) if every cell has a constant metric, else None.

        Uses the reference geometry arrays themselves (first quadrature point)
        so the constants are exactly the oracle's; constancy is checked."""
        geo, d, k = self.geometry, self.d, self.k
        if isinstance(geo, AffineGeometry):
            return geo.G, geo.det, geo.normal, geo.fscale
        E = self.mesh.n_elements
        if _is_tensor(geo.vol[k].inv_jac):
            # device geometry (precompute_geometry(device=...)): constancy test
            # on the device; only an affine mesh comes back to the host
            t = geo.vol[k].inv_jac.reshape(E, d, d, -1)
            t0 = t[..., :1]
            if float((t - t0).abs().max()) > rtol * max(float(t0.abs().max()), 1.0):
                return None
            geo = _host_geometry(geo)
        vol = geo.vol[k]
        ij = np.asarray(vol.inv_jac).reshape(E, d, d, -1)
        G = ij[..., 0]
        if np.max(np.abs(ij - G[..., None])) > rtol * max(np.max(np.abs(G)), 1.0):
            return None
        w = _lib.basis_table("gauss_weights", k)
        wt = w
        for _ in range(d - 1):
            wt = np.multiply.outer(w, wt)
        jr = np.asarray(vol.jxw).reshape(E, -1) / wt.ravel()[None, :]
        det = jr[:, 0]
        if np.max(np.abs(jr - det[:, None])) > rtol * np.max(np.abs(det)):
            return None
        wf = np.ones(()) if d == 1 else w
        for _ in range(d - 2):
            wf = np.multiply.outer(w, wf)
        normal = np.empty((E, d, 2, d))
        fscale = np.empty((E, d, 2))
        for m in range(d):
            for s in (0, 1):
                fg = geo.face[(m, s)]
                nr = np.asarray(fg.normal).reshape(E, d, -1)
                if np.max(np.abs(nr - nr[..., :1])) > rtol:
                    return None
                fj = np.asarray(fg.jxw).reshape(E, -1) / np.ravel(wf)[None, :]
                if np.max(np.abs(fj - fj[:, :1])) > rtol * np.max(np.abs(fj)):
                    return None
                normal[:, m, s] = nr[..., 0]
                fscale[:, m, s] = fj[:, 0] / det
        return G, det, normal, fscale

    def __del__(self):
        try:
            if self._ctx:
                lib().wk_ctx_destroy(self._ctx)
                self._ctx = ctypes.c_void_p()
        except Exception:
            pass

    # -- helpers ----------------------------------------------------------
    @property
    def stream(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def _check(self, state, basis: str = "gl") -> None:
        if state.basis != basis:
            raise ValueError(f"state must be in the {basis.upper()} basis")
        expect = (self.mesh.n_elements, self.n_comp) + (self.k + 1,) * self.d
        if tuple(state.data.shape) != expect:
            raise ValueError(f"state shape {tuple(state.data.shape)}, expected {expect}")

    def _dev(self, data):
        """(device tensor, was_numpy) for a numpy array or torch tensor."""
        torch = _torch()
        if isinstance(data, np.ndarray):
            host = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64))
            dev = torch.empty(host.shape, dtype=torch.float64, device=self.device)
            dev.copy_(host)
            return dev, True
        if data.dtype != torch.float64:
            raise ValueError("states must be float64")
        if data.device != self.device:
            data = data.to(self.device)
        return data.contiguous(), False

    @staticmethod
    def _ptr(t):
        return ctypes.c_void_p(t.data_ptr())

    def _out(self, t, was_np):
        """Device result back to numpy through a pinned staging buffer (the
        caching host allocator keeps it for the next call)."""
        if not was_np:
            return t
        torch = _torch()
        host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        host.copy_(t)
        return host.numpy()

    def new_state(self) -> StateVector:
        return StateVector.zeros(self.mesh.n_elements, self.k, self.d, device=self.device)

    def _unary(self, fn, data, shape=None, *extra):
        x, was_np = self._dev(data)
        torch = _torch()
        y = torch.empty(shape if shape is not None else x.shape, dtype=torch.float64,
                        device=self.device)
        check(fn(self._ctx, self._ptr(x), self._ptr(y), *extra, self.stream))
        return self._out(y, was_np)

    # -- derivative operator ----------------------------------------------
    def apply_K(self, state: StateVector, parts: str = "both") -> StateVector:
        self._check(state)
        if parts not in _lib.PARTS:
            raise ValueError(f"unknown parts {parts!r}")
        out = self._unary(lambda c, x, y, s: lib().wk_apply_K(c, x, y, _lib.PARTS[parts], s),
                          state.data)
        cost.count_apply_K(self.counter, self.mesh.n_elements, self.d, self.k, parts)
        return StateVector(out, self.k, self.d)

    def apply_minv_K(self, state: StateVector, parts: str = "both") -> StateVector:
        """M^{-1} K u in one fused kernel (apply_inverse_mass(apply_K(u)))."""
        self._check(state)
        out = self._unary(lambda c, x, y, s: lib().wk_apply_minv_K(c, x, y, _lib.PARTS[parts], s),
                          state.data)
        cost.count_apply_K(self.counter, self.mesh.n_elements, self.d, self.k, parts)
        cost.count_mass(self.counter, self.mesh.n_elements, self.d, self.k)
        return StateVector(out, self.k, self.d)

    def apply_inverse_mass(self, state: StateVector) -> StateVector:
        self._check(state)
        cost.count_mass(self.counter, self.mesh.n_elements, self.d, self.k)
        return StateVector(self._unary(lib().wk_apply_inverse_mass, state.data), self.k, self.d)

    def apply_mass(self, state: StateVector) -> StateVector:
        self._check(state)
        cost.count_mass(self.counter, self.mesh.n_elements, self.d, self.k)
        return StateVector(self._unary(lib().wk_apply_mass, state.data), self.k, self.d)

    def rhs(self, state: StateVector) -> StateVector:
        """-M^{-1} K u, fused (operator.py:268-272)."""
        self._check(state)
        cost.count_apply_K(self.counter, self.mesh.n_elements, self.d, self.k)
        cost.count_mass(self.counter, self.mesh.n_elements, self.d, self.k)
        return StateVector(self._unary(lib().wk_rhs, state.data), self.k, self.d)

    # -- collocated Taylor-loop operators -----------------------------------
    def to_gauss_values(self, data):
        self._count_sweeps(data.shape[0], self.k, self.k)
        return self._unary(lib().wk_to_gauss_values, data)

    def from_gauss_weighted(self, values):
        self._count_sweeps(values.shape[0], self.k, self.k)
        return self._unary(lib().wk_from_gauss_weighted, values)

    def _count_sweeps(self, E, q_from, q_to, phase="convert"):
        c = self.counter
        if c is not None and c.enabled:
            cost._sweeps(c, phase, E * self.n_comp, q_from + 1, q_to + 1, self.d)

    def apply_local_S(self, values, degree: int):
        if degree not in self._degrees():
            raise ValueError(f"geometry has no degree-{degree} point set; "
                             f"precompute it for this reduction policy")
        c = self.counter
        if c is not None and c.enabled:
            m = int(degree) + 1
            c.record("tck", units=values.shape[0] * self.n_comp * self.d, n_out=m, n_in=m,
                     lines=m ** (self.d - 1))
        return self._unary(lambda c, x, y, s: lib().wk_apply_local_S(c, x, y, int(degree), s),
                           values)

    def resize_values(self, values, k_from: int, k_to: int):
        if k_from == k_to:
            return values
        shape = tuple(values.shape[:2]) + (k_to + 1,) * self.d
        self._count_sweeps(values.shape[0], k_from, k_to)
        return self._unary(
            lambda c, x, y, s: lib().wk_resize_values(c, x, y, int(k_from), int(k_to), s),
            values, shape)
