"""Kernel-call counter and the reference's analytic cost model.

Mirrors ``/root/reference/pkg/src/wavekernel/kernels.py``: ``KernelCounter``
(:55-101), ``kernel_flops`` (:172-180), ``cost_tensorial`` (:183-188),
``kernel_call_table`` (:191-208), ``CostReport`` / ``scheme_cost``
(:211-279), ``reduction_schedule`` / ``reduction_degrees`` (:282-309) and
``tck_cost_model`` (:312-342), with the same signatures and numbers.

The reference counts FLOPs by recording every 1-D ``apply_1d`` call of its
numpy operator.  The GPU operator runs fused kernels that do far fewer
sweeps, so the counter here is fed the calls the REFERENCE
operator would have made for the same method, element count and degree
(:func:`count_apply_K`, :func:`count_mass`, :func:`count_tck` ...).  That
keeps the harness's "counted FLOPs == model FLOPs" cross-check
(reference cli.py:245-254, tests/test_cli.py:95-104) meaningful for the
GPU operator: the model is the reference's, and the tally reproduces the
reference's own per-phase, per-call bookkeeping (pinned against the
reference counter in tests/test_cost.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

__all__ = [
    "KernelCounter", "kernel_flops", "cost_tensorial", "kernel_call_table", "CostReport",
    "scheme_cost", "tck_cost_model", "reduction_schedule", "reduction_degrees",
    "REDUCTION_STRIDE", "count_apply_K", "count_mass", "count_tck", "count_scheme_step",
]

REDUCTION_STRIDE = {"none": 0, "every_step": 1, "every_second": 2, "every_third": 3}
_RK_STAGES = {"rk4_classic": 4, "lsrk45": 5, "lsrk59": 9}


class KernelCounter:
    """Per-phase tally of 1-D kernel calls and model FLOPs (kernels.py:55-101).

    Off by default; ``record`` is a no-op unless ``enabled``."""

    def __init__(self):
        self.enabled = False
        self.counts: dict[str, dict[str, int]] = {}

    def _bucket(self, phase: str) -> dict[str, int]:
        return self.counts.setdefault(phase, {"cell_calls": 0, "face_calls": 0, "flops": 0})

    def record(self, phase: str, *, units: int, n_out: int, n_in: int, lines: int,
               face: bool = False) -> None:
        if not self.enabled:
            return
        b = self._bucket(phase)
        b["face_calls" if face else "cell_calls"] += units
        b["flops"] += units * kernel_flops(n_out, n_in, lines)

    def reset(self) -> None:
        self.counts = {}

    def merge(self, other: "KernelCounter") -> None:
        for phase, ob in other.counts.items():
            b = self._bucket(phase)
            for key, val in ob.items():
                b[key] += val

    def calls(self, phase: str, face: bool = False) -> int:
        b = self.counts.get(phase)
        return 0 if b is None else b["face_calls" if face else "cell_calls"]

    def total_flops(self) -> int:
        return sum(b["flops"] for b in self.counts.values())


def kernel_flops(n_out: int, n_in: int, lines: int) -> int:
    """Model FLOPs of one 1-D call on ``lines`` lines, even-odd counting
    (kernels.py:172-180)."""
    return (3 * n_out + 2 * ((max(n_in - 2, 0) * n_out) // 2)) * lines


def cost_tensorial(k: int, delta: int) -> int:
    """One square call at degree k on a delta-dimensional tensor (kernels.py:183-188)."""
    if k < 1 or delta < 1:
        raise ValueError("need k >= 1 and delta >= 1")
    n = k + 1
    return kernel_flops(n, n, n ** (delta - 1))


def kernel_call_table(k: int, d: int) -> dict[str, dict[str, int]]:
    """Calls per element per scalar field of each operator (kernels.py:191-208)."""
    if d not in (2, 3):
        raise ValueError("call table is defined for d in {2, 3}")
    return {
        "mass": {"cell": 2 * d, "face": 0},
        "stiffness": {"cell": d * d + 4 * d, "face": 4 * (d * d - d)},
        "tck": {"cell": 2 * d + d * (k - 1), "face": 0},
    }


@dataclass(frozen=True)
class CostReport:
    """Model FLOPs per element per step, whole (d+1)-field system (kernels.py:211-229)."""

    scheme: str
    k: int
    d: int
    stages: int
    c_mass: int
    c_stiffness: int
    c_tck: int
    c_basis_change: int
    c_scheme_total: int
    calls: dict = field(default_factory=dict)


def scheme_cost(k: int, d: int, scheme: str, stages: int | None = None) -> CostReport:
    """Per-element per-step model FLOPs of a scheme (kernels.py:235-279)."""
    table = kernel_call_table(k, d)
    comps = d + 1
    cell, face = cost_tensorial(k, d), cost_tensorial(k, d - 1)
    c_mass = comps * table["mass"]["cell"] * cell
    c_stiff = comps * (table["stiffness"]["cell"] * cell + table["stiffness"]["face"] * face)
    c_tck = comps * table["tck"]["cell"] * cell
    c_conv = comps * 2 * d * cell
    if scheme in ("ader", "ader_hdg"):
        total = 2 * c_mass + c_stiff + c_tck
        if scheme == "ader_hdg":
            total += c_mass + c_stiff       # W = M^{-1} K U
        s = 0
    elif scheme == "rk" or scheme in _RK_STAGES:
        s = _RK_STAGES.get(scheme, stages)
        if s is None:
            raise ValueError("rk scheme needs a stage count")
        total = s * (c_mass + c_stiff)
        c_tck = c_conv = 0
    else:
        raise ValueError(f"unknown scheme {scheme!r}")
    return CostReport(scheme=scheme, k=k, d=d, stages=s, c_mass=c_mass, c_stiffness=c_stiff,
                      c_tck=c_tck, c_basis_change=c_conv, c_scheme_total=total, calls=table)


def reduction_schedule(k: int, policy: str) -> list[tuple[int, int]]:
    """(deg_in, deg_out) of each Taylor application (kernels.py:286-302)."""
    if policy not in REDUCTION_STRIDE:
        raise ValueError(f"unknown reduction policy {policy!r}")
    s, deg, out = REDUCTION_STRIDE[policy], k, []
    for j in range(1, k + 2):
        nxt = max(deg - s, 0) if (s and j % s == 0) else deg
        out.append((deg, nxt))
        deg = nxt
    return out


def reduction_degrees(k: int, policy: str) -> tuple[int, ...]:
    """Reduced degrees (< k, descending) a policy visits (kernels.py:305-309)."""
    return tuple(sorted({o for _, o in reduction_schedule(k, policy)} - {k}, reverse=True))


def _resize_cost(n_from: int, n_to: int, d: int) -> int:
    return sum(kernel_flops(n_to, n_from, n_to ** t * n_from ** (d - 1 - t)) for t in range(d))


def tck_cost_model(k: int, d: int, policy: str = "none") -> int:
    """Model FLOPs of one Taylor evaluation with the policy's extent schedule
    (kernels.py:312-342)."""
    n = k + 1
    per = 2 * d * kernel_flops(n, n, n ** (d - 1))
    accs = {k}
    for d_in, d_out in reduction_schedule(k, policy):
        m = d_in + 1
        per += d * kernel_flops(m, m, m ** (d - 1))
        if d_out != d_in:
            per += _resize_cost(d_in + 1, d_out + 1, d)
        accs.add(d_out)
    chain = sorted(accs)
    for lo, hi in zip(chain[:-1], chain[1:]):
        per += _resize_cost(lo + 1, hi + 1, d)
    return (d + 1) * per


# ---------------------------------------------------------------------------
# the reference operator's call bookkeeping, per method (operator.py:136-325)

def _sweeps(counter, phase, units, n_from, n_to, d, directions=None, face=False):
    """One _sweep (operator.py:136-142): a call per direction, extents
    changing direction by direction for a rectangular matrix."""
    span = d if directions is None else directions
    for t in range(span):
        counter.record(phase, units=units, n_out=n_to, n_in=n_from,
                       lines=n_to ** t * n_from ** (span - 1 - t), face=face)


def count_apply_K(counter, E: int, d: int, k: int, parts: str = "both", times: int = 1):
    """apply_K (operator.py:149-246): (d^2+4d) cell calls, 4(d^2-d) face
    calls per element and field (kernels.py:205)."""
    if counter is None or not counter.enabled:
        return
    n, units = k + 1, E * (d + 1) * times
    if parts in ("both", "cell"):
        counter.record("stiffness", units=units * (d * d + 4 * d), n_out=n, n_in=n,
                       lines=n ** (d - 1))
    if parts in ("both", "face"):
        counter.record("stiffness", units=units * 4 * (d * d - d), n_out=n, n_in=n,
                       lines=n ** (d - 2), face=True)


def count_mass(counter, E: int, d: int, k: int, times: int = 1):
    """apply_inverse_mass / apply_mass (operator.py:250-266): 2d calls."""
    if counter is None or not counter.enabled:
        return
    n = k + 1
    counter.record("mass", units=E * (d + 1) * 2 * d * times, n_out=n, n_in=n,
                   lines=n ** (d - 1))


def count_tck(counter, E: int, d: int, k: int, policy: str, shift: bool, times: int = 1):
    """tck_evaluate (stepping.py:215-262) through the operator's
    to_gauss_values / apply_local_S / resize_values / from_gauss_weighted."""
    if counter is None or not counter.enabled:
        return
    units = E * (d + 1) * times
    n = k + 1
    _sweeps(counter, "convert", units, n, n, d)                      # to_gauss_values
    sched = reduction_schedule(k, policy)
    n_apps = max(k - 1, 0) if shift else k + 1
    deg, accs = k, {k}
    for j in range(1, n_apps + 1):
        d_in, d_out = sched[j - 1]
        if d_in == 0:
            break
        m = deg + 1
        counter.record("tck", units=units * d, n_out=m, n_in=m, lines=m ** (d - 1))
        if d_out != d_in:
            _sweeps(counter, "convert", units, d_in + 1, d_out + 1, d)
            deg = d_out
        accs.add(deg)
    chain = sorted(accs)
    for lo, hi in zip(chain[:-1], chain[1:]):
        _sweeps(counter, "convert", units, lo + 1, hi + 1, d)
    _sweeps(counter, "convert", units, n, n, d)                      # from_gauss_weighted


def count_scheme_step(counter, scheme: str, E: int, d: int, k: int,
                      policy: str = "every_second", steps: int = 1):
    """One step of a fused scheme, as the reference's composed step counts it
    (stepping.py:163-285)."""
    if counter is None or not counter.enabled or steps <= 0:
        return
    if scheme in ("lsrk45", "lsrk59", "rk4"):
        s = {"lsrk45": 5, "lsrk59": 9, "rk4": 4}[scheme] * steps
        count_apply_K(counter, E, d, k, times=s)
        count_mass(counter, E, d, k, times=s)
    elif scheme == "ader":
        count_tck(counter, E, d, k, policy, False, times=steps)
        count_apply_K(counter, E, d, k, times=steps)
        count_mass(counter, E, d, k, times=2 * steps)
    elif scheme == "ader_hdg":
        count_apply_K(counter, E, d, k, times=2 * steps)
        count_mass(counter, E, d, k, times=3 * steps)
        count_tck(counter, E, d, k, policy, True, times=steps)
    else:
        raise ValueError(f"unknown scheme {scheme!r}")
