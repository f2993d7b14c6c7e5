"""Golden fixtures for the cost model, the kernel-call counter and the CLI,
made by running the UNMODIFIED reference (importable only in the build
container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cost.py

Writes ``tests/golden/cost.json``:
* ``scheme_cost`` / ``tck_cost_model`` / ``kernel_call_table`` numbers for
  d in {2, 3}, k = 1..12, every scheme and reduction policy
  (reference kernels.py:191-342);
* the reference operator's KernelCounter tallies per method on small meshes
  (apply_K per parts, inverse mass, mass, rhs, tck_evaluate per policy and
  shift, one step of every scheme) — what the GPU operator's counter
  emulation must reproduce (paper_1805_03981_b200/cost.py);
* the reference ``opcount`` table text (cli.py:247-276);
* reference ``run`` records (l2_err) for small 2-D cases, for the GPU CLI;
* reference ``hdg_flux`` (operator.py:70-87) on seeded pointwise inputs.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from wavekernel import cli as RC  # noqa: E402
from wavekernel.analytic import initial_state  # noqa: E402
from wavekernel.kernels import (kernel_call_table, reduction_degrees, scheme_cost,  # noqa: E402
                                tck_cost_model)
from wavekernel.mesh import Material, build_cartesian, deform, precompute_geometry  # noqa: E402
from wavekernel.operator import AcousticOperator  # noqa: E402
from wavekernel.stepping import SchemeConfig, make_stepper, tck_evaluate  # noqa: E402

POLICIES = ("none", "every_step", "every_second", "every_third")
SCHEMES = ("rk4_classic", "lsrk45", "lsrk59", "ader", "ader_hdg")


def model():
    out = {}
    for d in (2, 3):
        for k in range(1, 13):
            key = f"{d}_{k}"
            out[key] = {
                "table": kernel_call_table(k, d),
                "schemes": {s: {f: getattr(scheme_cost(k, d, s), f) for f in
                                ("stages", "c_mass", "c_stiffness", "c_tck", "c_basis_change",
                                 "c_scheme_total")} for s in SCHEMES},
                "tck": {p: tck_cost_model(k, d, p) for p in POLICIES},
            }
    return out


def counts():
    out = []
    for d, k, n, deform_amp in ((2, 3, 3, 0.0), (3, 2, 2, 0.0), (2, 5, 2, 0.1), (3, 4, 2, 0.0)):
        mesh = build_cartesian(n, d, "periodic")
        if deform_amp:
            mesh = deform(mesh, deform_amp)
        mat = Material.uniform(mesh)
        degs = sorted(set(sum((reduction_degrees(k, p) for p in POLICIES), ())))
        geo = precompute_geometry(mesh, k, reduced_degrees=tuple(degs))
        op = AcousticOperator(mesh, geo, mat)
        st = initial_state(mesh, k, mat, m=1)
        c = op.counter
        case = {"d": d, "k": k, "elements": mesh.n_elements, "deform": deform_amp, "calls": {}}

        def tally(name, fn):
            c.reset()
            c.enabled = True
            fn()
            c.enabled = False
            case["calls"][name] = {ph: dict(v) for ph, v in c.counts.items()}

        for parts in ("both", "cell", "face"):
            tally(f"apply_K:{parts}", lambda: op.apply_K(st, parts))
        tally("apply_inverse_mass", lambda: op.apply_inverse_mass(st))
        tally("apply_mass", lambda: op.apply_mass(st))
        tally("rhs", lambda: op.rhs(st))
        for p in POLICIES:
            for shift in (False, True):
                tally(f"tck:{p}:{int(shift)}", lambda: tck_evaluate(st, 1e-3, op, p, shift=shift))
        for s in ("rk4", "lsrk45", "lsrk59", "ader", "ader_hdg"):
            for p in ("none", "every_second"):
                if s.startswith(("rk", "lsrk")) and p != "none":
                    continue
                step = make_stepper(SchemeConfig(scheme=s, degree_reduction=p), op)
                tally(f"step:{s}:{p}", lambda: step(st, 1e-3))
        out.append(case)
    return out


def opcount_text():
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        RC.main(["opcount"])
    return buf.getvalue()


def run_records():
    recs = []
    for args in (["run", "--degree", "3", "--elements", "4", "--scheme", "lsrk45",
                  "--end-time", "0.25"],
                 ["run", "--degree", "2", "--elements", "4", "--scheme", "ader-hdg",
                  "--end-time", "0.25", "--boundary", "periodic", "--mode", "2"],
                 ["run", "--degree", "3", "--elements", "4", "--scheme", "ader",
                  "--end-time", "0.125", "--reduction", "none"],
                 ["run", "--degree", "2", "--elements", "4", "--scheme", "lsrk59",
                  "--end-time", "0.125", "--deform", "0.05"]):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert RC.main(args) == 0
        lines = buf.getvalue().strip().splitlines()
        rec = dict(zip(lines[0].split(","), lines[1].split(",")))
        recs.append({"args": args, "steps": int(rec["steps"]), "l2_err": float(rec["l2_err"]),
                     "model_flops": int(rec["model_flops"]), "dofs": int(rec["dofs"])})
    return recs


def flux_cases():
    """reference hdg_flux (operator.py:70-87) on seeded pointwise inputs"""
    from wavekernel.operator import hdg_flux
    import numpy as np
    out = []
    for d, tau, seed in ((2, None, 0), (3, 0.7, 1), (3, 0.0, 2), (2, 1.3, 3)):
        rng = np.random.default_rng(seed)
        vm, vp = rng.standard_normal((d, 5)), rng.standard_normal((d, 5))
        pm, pp = rng.standard_normal(5), rng.standard_normal(5)
        nrm = rng.standard_normal((d, 5))
        nrm /= np.linalg.norm(nrm, axis=0)
        c, rho = float(rng.uniform(0.5, 2)), float(rng.uniform(0.5, 2))
        fv, fp = hdg_flux((vm, pm), (vp, pp), nrm, c, rho, tau)
        out.append({"d": d, "tau": tau, "c": c, "rho": rho, "vm": vm.tolist(), "vp": vp.tolist(),
                    "pm": pm.tolist(), "pp": pp.tolist(), "n": nrm.tolist(),
                    "fv": fv.tolist(), "fp": fp.tolist()})
    return out


if __name__ == "__main__":
    payload = {"model": model(), "counts": counts(), "opcount": opcount_text(),
               "run": run_records(), "hdg_flux": flux_cases()}
    with open(os.path.join(HERE, "cost.json"), "w") as fh:
        json.dump(payload, fh, indent=0, sort_keys=True)
        fh.write("\n")
    print("wrote cost.json")
