"""GPU drop-in for the reference time integrators.

Mirrors ``/root/reference/pkg/src/wavekernel/stepping.py``: the scheme
tables (``LSRK45`` :88-106, ``LSRK59`` :113-143, ``RK4_CLASSIC`` :57-64),
``SchemeConfig`` (:148-160), ``rk_step`` (:163-176), ``lsrk_step``
(:179-207), ``tck_evaluate`` (:215-262), ``ader_step`` (:265-285),
``make_stepper`` (:288-302), ``advance`` (:305-308), ``compute_dt``
(:311-318) and ``state_norm`` (:321-324), with the same signatures.

With the GPU :class:`AcousticOperator` the steppers run the fused kernels:
one kernel per LSRK stage (operator + inverse mass + register update), two
kernels per ADER step.  With any other duck-typed operator (e.g. a counting
proxy, as in the reference's tests) they compose the operator's public
methods exactly like the reference does.

Deviation (documented in DESIGN.md): the fused LSRK keeps THREE state
vectors on the device (u ping-pong + r), not the reference's two, because a
stage reads neighbour faces of u while other elements are already writing
their update.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib, cost
from .cost import reduction_degrees, reduction_schedule
from ._lib import check, lib
from .mesh import min_edge_length
from .operator import AcousticOperator, StateVector

__all__ = [
    "ButcherTableau", "RK4_CLASSIC", "LowStorageScheme", "LSRK45", "LSRK59",
    "SchemeConfig", "rk_step", "lsrk_step", "tck_evaluate", "ader_step",
    "advance", "compute_dt", "state_norm", "make_stepper", "DeviceStepper",
    "SCHEME_STAGES", "reduction_schedule", "reduction_degrees", "CourantSearchError",
    "find_critical_courant",
]


@dataclass(frozen=True)
class ButcherTableau:
    a: tuple
    b: tuple
    c: tuple

    @property
    def stages(self) -> int:
        return len(self.b)


RK4_CLASSIC = ButcherTableau(
    a=((0.0, 0.0, 0.0, 0.0), (0.5, 0.0, 0.0, 0.0), (0.0, 0.5, 0.0, 0.0), (0.0, 0.0, 1.0, 0.0)),
    b=(1 / 6, 1 / 3, 1 / 3, 1 / 6),
    c=(0.0, 0.5, 0.5, 1.0),
)


@dataclass(frozen=True)
class LowStorageScheme:
    name: str
    a: tuple
    b: tuple
    c: tuple
    order: int

    def __post_init__(self):
        if not (len(self.a) == len(self.b) == len(self.c)):
            raise ValueError("coefficient arrays disagree in length")
        if self.a[0] != 0.0:
            raise ValueError("first register weight must vanish")

    @property
    def stages(self) -> int:
        return len(self.b)


# Carpenter & Kennedy (1994) 2N five-stage fourth-order coefficients
LSRK45 = LowStorageScheme(
    name="lsrk45",
    a=(0.0, -567301805773 / 1357537059087, -2404267990393 / 2016746695238,
       -3550918686646 / 2091501179385, -1275806237668 / 842570457699),
    b=(1432997174477 / 9575080441755, 5161836677717 / 13612068292357,
       1720146321549 / 2090206949498, 3134564353537 / 4481467310338,
       2277821191437 / 14882151754819),
    c=(0.0, 1432997174477 / 9575080441755, 2526269341429 / 6820363962896,
       2006345519317 / 3224310063776, 2802321613138 / 2924317926251),
    order=4,
)

# The reference's nine-stage register weights (stepping.py:113-143)
LSRK59 = LowStorageScheme(
    name="lsrk59",
    a=(0.0, -0.6304365496865543, -1.1303843359562102, -0.3293878463661334,
       -1.4487682419993357, -0.8130202966406633, -0.9436317245996502,
       -0.058029253696775494, -1.2209100426892907),
    b=(0.03321496462492457, 0.5563858748215249, 0.721229659783645, 0.0770373034268954,
       0.7269522462792919, 0.27832474096203197, 0.19393254670497226,
       0.16876385757079637, 0.304085932161835),
    c=(0.0, 0.03321496462492457, 0.23883484822963222, 0.6587717297228163,
       0.7210343191188239, 0.5967879549918808, 0.9137877569225696, 0.8992902159424159,
       1.0687861729512562),
    order=5,
)

SCHEME_STAGES = {"rk4": 4, "lsrk45": 5, "lsrk59": 9}
_STRIDE = {"none": 0, "every_step": 1, "every_second": 2, "every_third": 3}


@dataclass
class SchemeConfig:
    scheme: str = "lsrk45"
    courant: float = 0.3
    degree_reduction: str = "every_second"
    merged_vector_update: bool = True

    def __post_init__(self):
        known = ("rk4", "lsrk45", "lsrk59", "ader", "ader_hdg")
        if self.scheme not in known:
            raise ValueError(f"unknown scheme {self.scheme!r}; choose one of {known}")


def _fused(op) -> bool:
    return type(op) is AcousticOperator


def _like(data, arr):
    return arr


def _new_like(x):
    if isinstance(x, np.ndarray):
        return np.zeros_like(x)
    return x.new_zeros(x.shape)


# ---------------------------------------------------------------------------
def rk_step(state: StateVector, dt: float, tableau: ButcherTableau, op) -> StateVector:
    """Classical stage-storage RK step (reference quality, composed)."""
    ks = []
    for i in range(tableau.stages):
        y = state.data
        for j, aij in enumerate(tableau.a[i][:i]):
            if aij != 0.0:
                y = y + dt * aij * ks[j]
        ks.append(op.rhs(StateVector(y, state.degree, state.dim)).data)
    out = state.data.copy() if isinstance(state.data, np.ndarray) else state.data.clone()
    for bj, kj in zip(tableau.b, ks):
        out = out + dt * bj * kj
    return StateVector(out, state.degree, state.dim)


def lsrk_step(state: StateVector, dt: float, scheme: LowStorageScheme, op,
              merged: bool = True, alloc_hook=None) -> StateVector:
    """One low-storage RK step (stepping.py:179-207).

    GPU operator: each stage is ONE fused kernel (f = -M^{-1}Ku, r = a r +
    dt f, u' = u + b r) over three device vectors (see module doc)."""
    if _fused(op):
        op._check(state)
        x, was_np = op._dev(state.data)
        u = x.clone() if not was_np else x
        if alloc_hook is not None:
            alloc_hook(u.numel() * 8)
        u2 = u.new_empty(u.shape)
        if alloc_hook is not None:
            alloc_hook(u2.numel() * 8)
        r = u.new_empty(u.shape)
        if alloc_hook is not None:
            alloc_hook(r.numel() * 8)
        s = op.stream
        cost.count_apply_K(op.counter, op.mesh.n_elements, op.d, op.k, times=scheme.stages)
        cost.count_mass(op.counter, op.mesh.n_elements, op.d, op.k, times=scheme.stages)
        for i, (a, b) in enumerate(zip(scheme.a, scheme.b)):
            # r is local to the step (stepping.py:184-195): dead after the last stage
            check(lib().wk_lsrk_stage_ex(op._ctx, op._ptr(u), op._ptr(u2), op._ptr(r),
                                         float(a), float(b), float(dt),
                                         int(i == scheme.stages - 1), s))
            u, u2 = u2, u
        return StateVector(op._out(u, was_np), state.degree, state.dim)
    # composed path through the duck-typed operator (reference arithmetic)
    u = state.data.copy() if isinstance(state.data, np.ndarray) else state.data.clone()
    if alloc_hook is not None:
        alloc_hook(u.nbytes if isinstance(u, np.ndarray) else u.numel() * 8)
    r = _new_like(u)
    if alloc_hook is not None:
        alloc_hook(r.nbytes if isinstance(r, np.ndarray) else r.numel() * 8)
    for a, b in zip(scheme.a, scheme.b):
        f = op.rhs(StateVector(u, state.degree, state.dim)).data
        r = r * a + f * dt
        u = u + r * b
    return StateVector(u, state.degree, state.dim)


def _taylor_weight(j: int, dt: float) -> float:
    return (-1.0 if j % 2 else 1.0) * dt ** (j + 1) / math.factorial(j + 1)


def tck_evaluate(state: StateVector, dt: float, op, reduction: str = "every_second",
                 shift: bool = False) -> StateVector:
    """Element-local Taylor sum, mass-weighted GL output (stepping.py:215-262)."""
    op._check(state)
    if reduction not in _STRIDE:
        raise ValueError(f"unknown reduction policy {reduction!r}")
    k = state.degree
    if _fused(op):
        x, was_np = op._dev(state.data)
        out = x.new_empty(x.shape)
        cost.count_tck(op.counter, op.mesh.n_elements, op.d, k, reduction, shift)
        check(lib().wk_tck(op._ctx, op._ptr(x), op._ptr(out), float(dt),
                           _lib.POLICY[reduction], 1 if shift else 0, op.stream))
        return StateVector(op._out(out, was_np), k, state.dim)
    cur = op.to_gauss_values(state.data)
    acc = {k: _taylor_weight(1 if shift else 0, dt) * cur}
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
        w = _taylor_weight(j + 1 if shift else j, dt)
        acc[deg] = acc[deg] + w * cur if deg in acc else w * cur
    for lo in sorted(acc):
        if lo == k:
            break
        hi = min(q for q in acc if q > lo)
        acc[hi] = acc[hi] + op.resize_values(acc[lo], lo, hi)
    return StateVector(op.from_gauss_weighted(acc[k]), k, state.dim)


def ader_step(state: StateVector, dt: float, op, variant: str = "ader_hdg",
              reduction: str = "every_second") -> StateVector:
    """One ADER step (stepping.py:265-285); two fused kernels on the GPU."""
    if variant not in ("ader", "ader_hdg"):
        raise ValueError(f"unknown ader variant {variant!r}")
    if _fused(op):
        op._check(state)
        x, was_np = op._dev(state.data)
        U = x.clone() if not was_np else x
        Y = U.new_empty(U.shape)
        V = U.new_empty(U.shape) if variant == "ader_hdg" else None
        cost.count_scheme_step(op.counter, variant, op.mesh.n_elements, op.d, op.k, reduction)
        check(lib().wk_ader_step(op._ctx, _lib.WK_ADER_HDG if variant == "ader_hdg"
                                 else _lib.WK_ADER, _lib.POLICY[reduction], op._ptr(U),
                                 op._ptr(V) if V is not None else None, op._ptr(Y),
                                 float(dt), op.stream))
        return StateVector(op._out(U, was_np), state.degree, state.dim)
    if variant == "ader":
        t = tck_evaluate(state, dt, op, reduction=reduction)
        z = op.apply_inverse_mass(op.apply_K(op.apply_inverse_mass(t)))
        return StateVector(state.data - z.data, state.degree, state.dim)
    w = op.apply_inverse_mass(op.apply_K(state))
    t = tck_evaluate(w, dt, op, reduction=reduction, shift=True)
    z = op.apply_inverse_mass(op.apply_K(op.apply_inverse_mass(t)))
    return StateVector(state.data - dt * w.data - z.data, state.degree, state.dim)


class DeviceStepper:
    """Persistent-buffer stepper for the GPU operator.

    ``make_stepper`` returns one; calling it is the reference's
    ``(state, dt) -> state`` closure, and :func:`advance` recognises it and
    runs all steps on resident device buffers without per-step copies."""

    def __init__(self, config: SchemeConfig, op: AcousticOperator):
        self.config = config
        self.op = op
        self.name = config.scheme
        if self.name not in ("lsrk45", "lsrk59", "ader", "ader_hdg"):
            raise ValueError(f"no fused device stepper for {self.name!r}")
        self.scheme = LSRK45 if self.name == "lsrk45" else LSRK59
        self._bufs = None
        self._state = None
        self._graph = None      # (key, CUDAGraph) replaying GRAPH_STEPS steps
        self.use_graph = True

    def __call__(self, state: StateVector, dt: float) -> StateVector:
        return advance(state, dt, 1, self)

    def buffers(self, u):
        if self._bufs is None or self._bufs[0].shape != u.shape:
            self._bufs = (u.new_empty(u.shape), u.new_empty(u.shape))
        return self._bufs

    def state_buffer(self, shape):
        """Persistent device vector for host (numpy) states."""
        import torch
        if self._state is None or tuple(self._state.shape) != tuple(shape):
            self._state = torch.empty(tuple(shape), dtype=torch.float64, device=self.op.device)
        return self._state

    def launches_per_step(self) -> int:
        return self.scheme.stages if self.name.startswith("lsrk") else 2

    def _eager(self, u, dt: float, n_steps: int):
        op, s = self.op, self.op.stream
        ctx, P = op._ctx, op._ptr
        if self.name.startswith("lsrk") and getattr(op, "small_run", False):
            # the whole run in one thread-block-cluster launch, in place
            st = self.scheme.stages
            a = (ctypes.c_double * st)(*self.scheme.a)
            b = (ctypes.c_double * st)(*self.scheme.b)
            check(lib().wk_lsrk_run(ctx, P(u), P(u), st, a, b, float(dt), int(n_steps), s))
            return u
        b1, b2 = self.buffers(u)
        if self.name.startswith("lsrk"):
            cur, nxt, r = u, b1, b2
            for _ in range(n_steps):
                last = self.scheme.stages - 1
                for i, (a, b) in enumerate(zip(self.scheme.a, self.scheme.b)):
                    # the next step's first stage has a = 0: r is dead after the last
                    check(lib().wk_lsrk_stage_ex(ctx, P(cur), P(nxt), P(r), float(a), float(b),
                                                 float(dt), int(i == last), s))
                    cur, nxt = nxt, cur
            return cur
        variant = _lib.WK_ADER_HDG if self.name == "ader_hdg" else _lib.WK_ADER
        pol = _lib.POLICY[self.config.degree_reduction]
        for _ in range(n_steps):
            check(lib().wk_ader_step(ctx, variant, pol, P(u), P(b1), P(b2), float(dt), s))
        return u

    # two steps bring an odd-stage LSRK ping-pong back to `u`; ADER is in place
    GRAPH_STEPS = 2

    def _key(self, u, dt):
        return (u.data_ptr(), float(dt), tuple(u.shape))

    def capture(self, u, dt: float):
        """Record the CUDA graph of GRAPH_STEPS steps on ``u`` with this dt
        (recording runs nothing).  At least one eager step with this dt must
        have run before, so that one-time setup (function attributes, Taylor
        weights) is not captured."""
        import torch
        key = self._key(u, dt)
        if self._graph is None or self._graph[0] != key:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._eager(u, dt, self.GRAPH_STEPS)
            self._graph = (key, g)
        return self._graph[1]

    def run(self, u, dt: float, n_steps: int):
        """Advance the device tensor ``u`` n_steps; returns the tensor holding
        the result (``u`` or an internal buffer).

        Long runs replay a CUDA graph of GRAPH_STEPS steps (captured once per
        (buffer, dt)); the first steps run eagerly, which also performs every
        one-time setup (function attributes, Taylor weights) outside capture."""
        op = self.op
        cost.count_scheme_step(op.counter, self.name, op.mesh.n_elements, op.d, op.k,
                               self.config.degree_reduction, steps=n_steps)
        G = self.GRAPH_STEPS
        have = self._graph is not None and self._graph[0] == self._key(u, dt)
        if self.name.startswith("lsrk") and getattr(op, "small_run", False):
            return self._eager(u, dt, n_steps)     # one launch already
        if not self.use_graph or (not have and n_steps < 3 * G):
            return self._eager(u, dt, n_steps)
        done = 0
        if not have:
            res = self._eager(u, dt, G)          # warm-up, result back in u
            assert res is u
            done = G
        g = self.capture(u, dt)
        while n_steps - done >= G:
            g.replay()
            done += G
        return self._eager(u, dt, n_steps - done) if done < n_steps else u


def make_stepper(config: SchemeConfig, op):
    """Bind a config to a ``(state, dt)`` closure (stepping.py:288-302)."""
    name = config.scheme
    if _fused(op) and name != "rk4":
        return DeviceStepper(config, op)
    if name == "rk4":
        return lambda s, dt: rk_step(s, dt, RK4_CLASSIC, op)
    if name == "lsrk45":
        return lambda s, dt: lsrk_step(s, dt, LSRK45, op, merged=config.merged_vector_update)
    if name == "lsrk59":
        return lambda s, dt: lsrk_step(s, dt, LSRK59, op, merged=config.merged_vector_update)
    if name in ("ader", "ader_hdg"):
        return lambda s, dt: ader_step(s, dt, op, variant=name,
                                       reduction=config.degree_reduction)
    raise ValueError(f"unknown scheme {name!r}")


def advance(state: StateVector, dt: float, n_steps: int, stepper) -> StateVector:
    """Apply ``stepper`` n_steps times (stepping.py:305-308)."""
    if isinstance(stepper, DeviceStepper):
        op = stepper.op
        op._check(state)
        if isinstance(state.data, np.ndarray):
            # host state: one H2D into the stepper's persistent device vector
            # (so the recorded CUDA graph is reused across calls), K steps,
            # one D2H through a pinned staging buffer
            import torch
            u = stepper.state_buffer(state.data.shape)
            u.copy_(torch.from_numpy(np.ascontiguousarray(state.data, dtype=np.float64)))
            res = stepper.run(u, dt, n_steps)
            return StateVector(op._out(res, True), state.degree, state.dim)
        x, _ = op._dev(state.data)
        u = x.clone()
        res = stepper.run(u, dt, n_steps)
        if res is not u:
            # odd-stage LSRK with an odd eager step count ends in the
            # stepper's ping-pong buffer, which the next call overwrites: the
            # reference returns a fresh StateVector every time (stepping.py:305-308)
            u.copy_(res)
        return StateVector(u, state.degree, state.dim)
    for _ in range(n_steps):
        state = stepper(state, dt)
    return state


def compute_dt(courant: float, mesh, material, k: int) -> float:
    """dt = Cr h_min / (c_max k^1.5) (stepping.py:311-318)."""
    if courant <= 0.0:
        raise ValueError("Courant number must be positive")
    return courant * min_edge_length(mesh) / (float(np.max(material.c)) * max(k, 1) ** 1.5)


def state_norm(op, state: StateVector) -> float:
    """Mass-weighted discrete L2 norm (stepping.py:321-324).

    GPU operator: one fused kernel (wk_state_norm_sq, B sweeps + JxW-weighted
    squares + fixed-order reduction); other operators: the reference's
    composition through apply_mass."""
    if _fused(op):
        import ctypes
        import torch
        x, _ = op._dev(state.data)
        res = torch.empty(1, dtype=torch.float64, device=x.device)
        check(lib().wk_state_norm_sq(op._ctx, op._ptr(x), ctypes.c_void_p(res.data_ptr()),
                                     op.stream))
        return float(math.sqrt(abs(float(res.item()))))
    m = op.apply_mass(state)
    a, b = state.data, m.data
    if isinstance(a, np.ndarray):
        return float(np.sqrt(np.abs(np.vdot(a, b))))
    return float((a.reshape(-1) @ b.reshape(-1)).abs().sqrt())


class CourantSearchError(RuntimeError):
    """stepping.py:327-328"""


def find_critical_courant(config: SchemeConfig, mesh, k: int, scheme: str | None = None, *,
                          op=None, material=None, lo: float = 0.01, hi: float = 2.0,
                          width: float = 0.01, n_steps: int = 1000, mode: int = 1) -> float:
    """Bisect the largest stable Courant number to the given width
    (stepping.py:331-386), on the GPU.

    A run is stable when, after n_steps from the mode initial condition, the
    mass-weighted norm is finite and at most 10x its start; every 50 steps a
    norm above 1e6x the start (or non-finite) ends the run early.  The steps
    are the fused device stepper's CUDA-graph replays, the norm is the fused
    norm kernel and the initial state the mode kernel: the only host traffic
    is one scalar per 50 steps.  Raises CourantSearchError when the brackets
    do not straddle the stability boundary."""
    from .analytic import initial_state
    from .mesh import Material, precompute_geometry

    if scheme is not None:
        config = SchemeConfig(scheme=scheme, courant=config.courant,
                              degree_reduction=config.degree_reduction,
                              merged_vector_update=config.merged_vector_update)
    if material is None:
        material = Material.uniform(mesh)
    if op is None:
        geo = precompute_geometry(mesh, k, reduced_degrees=reduction_degrees(
            k, config.degree_reduction), device="cuda")
        op = AcousticOperator(mesh, geo, material)
    stepper = make_stepper(config, op)
    init = initial_state(mesh, k, material, m=mode)
    norm0 = state_norm(op, init)

    def stable(cr: float) -> bool:
        dt = compute_dt(cr, mesh, material, k)
        bound = 10.0 * norm0
        if isinstance(stepper, DeviceStepper):
            u = init.data.clone()
            done = 0
            while done < n_steps:
                chunk = min(50, n_steps - done)
                u = stepper.run(u, dt, chunk)
                done += chunk
                if chunk == 50:
                    nrm = state_norm(op, StateVector(u, k, mesh.d))
                    if not np.isfinite(nrm) or nrm > 1e6 * norm0:
                        return False
            nrm = state_norm(op, StateVector(u, k, mesh.d))
        else:
            u = init.copy()
            for i in range(n_steps):
                u = stepper(u, dt)
                if i % 50 == 49:
                    nrm = state_norm(op, u)
                    if not np.isfinite(nrm) or nrm > 1e6 * norm0:
                        return False
            nrm = state_norm(op, u)
        return bool(np.isfinite(nrm) and nrm <= bound)

    if not stable(lo):
        raise CourantSearchError(f"lower bracket Cr={lo} already unstable")
    if stable(hi):
        raise CourantSearchError(f"no unstable bracket found up to Cr={hi}")
    while hi - lo > width:
        mid = 0.5 * (lo + hi)
        if stable(mid):
            lo = mid
        else:
            hi = mid
    return lo
